O=gpurun_out/${1:-r02j}; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -k "1d or c4 or C4 or particle or ws_reuse or zero or lorenzo or secondary or smooth1d" > $O/pytest.log 2>&1
timeout 600 python bench.py --no-cpu --no-parity > $O/bench_c4.json 2> $O/bench_c4.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c4.csv python scripts/prof_roundtrip.py 280953867 default 1e-4 > $O/ncu_c4.log 2>&1
