#!/bin/bash
# Huffman decode sweeps: parity (Huffman / decode-error / full-size tests) + C4/C1 sweep times + C4 bench
O=gpurun_out/${1:-hfs}; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -k "huffman or decode or fullsize or parity or golden or secondary" > $O/tests.txt 2>&1; echo "tests exit $?" >> $O/tests.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"hf_sync" -c 8 --csv --log-file $O/l_c4.csv python scripts/prof_roundtrip.py 280953867 default 1e-4 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"hf_sync" -c 8 --csv --log-file $O/l_c1.csv python scripts/prof_roundtrip.py 100x500x500 default 1e-4 > /dev/null 2>&1
timeout 900 python bench.py --no-cpu > $O/bench_c4.json 2> $O/bench_c4.err
