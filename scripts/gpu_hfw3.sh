#!/bin/bash
O=gpurun_out/${1:-hfw3}; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/tests.txt 2>&1; echo "tests exit $?" >> $O/tests.txt
for c in "280953867 default 1e-4 c4" "100x500x500 default 1e-4 c1" "1800x3600 quality 1e-4 c3"; do set -- $c
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"hf_write_dec2" -c 2 --csv --log-file $O/l_$4.csv python scripts/prof_roundtrip.py $1 $2 $3 > /dev/null 2>&1
done
timeout 900 python bench.py --no-cpu --steps 5 > $O/bench_c4.json 2> $O/bench_c4.err
