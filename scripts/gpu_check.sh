# full GPU test suite + C4 bench + C4/C1 launch lists
O=gpurun_out/${1:-r02m}; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1
timeout 600 python bench.py --no-cpu --no-parity > $O/bench_c4.json 2> $O/bench_c4.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c4.csv python scripts/prof_roundtrip.py 280953867 default 1e-4 > $O/ncu_c4.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c1.csv python scripts/prof_roundtrip.py 100x500x500 default 1e-4 > $O/ncu_c1.log 2>&1
