O=gpurun_out/i2d9; mkdir -p $O
for v in 0 1 2 3; do
FZB_I2D=$v timeout 300 python bench.py --workload c3 --no-cpu > $O/bench_c3_v$v.json 2>&1
FZB_I2D=$v timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:interp2d -c 8 --csv --log-file $O/l_v$v.csv python bench.py --workload c3 --steps 2 --warmup 1 --no-cpu --no-parity > /dev/null 2>&1
done
