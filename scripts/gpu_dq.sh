O=gpurun_out/${1:-r02x}; mkdir -p $O
timeout 900 python -m pytest tests/test_dualquant.py -q -x -m gpu > $O/pytest_dq.log 2>&1
timeout 600 python bench.py --workload c2 --pipeline dq-speed --no-cpu > $O/bench_c2dq.json 2> $O/bench_c2dq.err
timeout 600 python bench.py --workload c2 --pipeline dq-default --no-cpu > $O/bench_c2dqd.json 2> $O/bench_c2dqd.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c2dq.csv python scripts/prof_roundtrip.py 512x512x512 dq-speed 1e-3 > $O/ncu_c2dq.log 2>&1
