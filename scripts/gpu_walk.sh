mkdir -p gpurun_out/r02e
export FZB_SO=paper_2509_20563_b200/_build/var/libfzb200_timing.so
for pf in 0 1024 4096; do echo "v6 2cta PF=$pf" >> gpurun_out/r02e/walk.txt; FZB_WALK_PF=$pf timeout 300 python scripts/walk_timing.py >> gpurun_out/r02e/walk.txt 2>&1; done
echo "v3 PF=0 twice" >> gpurun_out/r02e/walk.txt; FZB_WALK_TWICE=1 FZB_WALK_PF=0 timeout 300 python scripts/walk_timing.py >> gpurun_out/r02e/walk.txt 2>&1
echo "v3 1e-3" >> gpurun_out/r02e/walk.txt; timeout 300 python scripts/walk_timing.py 280953867 1e-3 >> gpurun_out/r02e/walk.txt 2>&1
unset FZB_SO
timeout 900 python -m pytest tests -m gpu -q -x -k "1d or c4 or C4 or particle or ws_reuse or zero or lorenzo" > gpurun_out/r02e/pytest.log 2>&1
timeout 600 python bench.py --workload c4 --no-cpu > gpurun_out/r02e/bench_c4.json 2> gpurun_out/r02e/bench_c4.err
