# One GPU session: the driver's bench invocations + the other workloads.
O=gpurun_out/${1:-r02h}; mkdir -p $O
timeout 900 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err
timeout 900 python bench.py --workload c5 --steps 3 --no-cpu > $O/bench_c5.json 2> $O/bench_c5.err
timeout 600 python bench.py --workload c2 --no-cpu > $O/bench_c2.json 2> $O/bench_c2.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref_c4.json 2> $O/bench_ref_c4.err
