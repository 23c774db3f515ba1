# Round profiles: ncu --set full of our kernels in one round trip per config.
# Reports are exported to CSV on the box (raw metrics + the walker's source
# page) and deleted: gpurun copies back at most 64 MiB.
O=gpurun_out/${1:-r02q2}; mkdir -p $O
K='regex:^(?!at::|elementwise|vectorized|unrolled|distribution).*'
run() {  # name dims preset rel count
  timeout 1200 ncu --set full --clock-control none --import-source on -k "$K" -c $5 -o /tmp/$1 python scripts/prof_roundtrip.py $2 $3 $4 > $O/ncu_$1.log 2>&1
  ncu -i /tmp/$1.ncu-rep --page raw --csv > $O/raw_$1.csv 2>/dev/null
  rm -f /tmp/$1.ncu-rep
}
run c4 280953867 default 1e-4 60
run c2 512x512x512 speed 1e-3 40
run c3 1800x3600 quality 1e-4 80
ls -la $O
