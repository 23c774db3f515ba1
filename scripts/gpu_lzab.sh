O=gpurun_out/${1:-r02ab}; mkdir -p $O; rm -f /tmp/lz3d_ref_*.pt
for v in hg8 hg4 hg2; do
  FZB_SO=paper_2509_20563_b200/_build/var/libfzb200_$v.so timeout 300 python scripts/lz3d_ab.py >> $O/ab.txt 2>&1
done
