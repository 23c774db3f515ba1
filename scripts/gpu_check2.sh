#!/bin/bash
# Parity suite + the single-field workloads + launch lists (C4, C1, 512^3 Default = a C5 field)
O=gpurun_out/${1:-chk}; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/tests.txt 2>&1; echo "tests exit $?" >> $O/tests.txt
for w in c4 c1 c2 c3; do timeout 900 python bench.py --workload $w --no-cpu > $O/bench_$w.json 2> $O/bench_$w.err; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c4.csv python scripts/prof_roundtrip.py 280953867 default 1e-4 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c1.csv python scripts/prof_roundtrip.py 100x500x500 default 1e-4 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c5f.csv python scripts/prof_roundtrip.py 512x512x512 default 1e-3 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c4s.csv python scripts/prof_roundtrip.py 280953867 speed 1e-4 > /dev/null 2>&1
