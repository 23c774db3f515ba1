#!/bin/bash
# 1D prepare/walk split: GPU suite + C4 bench + C4 launch list
O=gpurun_out/${1:-p1d}; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/tests.txt 2>&1; echo "tests exit $?" >> $O/tests.txt
timeout 900 python bench.py --no-cpu > $O/bench_c4.json 2> $O/bench_c4.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c4.csv python scripts/prof_roundtrip.py 280953867 default 1e-4 > /dev/null 2>&1
