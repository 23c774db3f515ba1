#!/bin/bash
# 1D decode chain: parity (1D tests + full-size C4) + launch times + C4 bench
O=gpurun_out/${1:-chain}; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -k "1d or fullsize or walker or particle or c4 or ws_reuse or golden" > $O/tests.txt 2>&1; echo "tests exit $?" >> $O/tests.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"lz1d" -c 20 --csv --log-file $O/l_c4.csv python scripts/prof_roundtrip.py 280953867 default 1e-4 > /dev/null 2>&1
timeout 900 python bench.py --no-cpu > $O/bench_c4.json 2> $O/bench_c4.err
