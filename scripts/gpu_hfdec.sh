#!/bin/bash
# Huffman decode write pass: parity (GPU suite subset) + C4/C1 bench + launch list
O=gpurun_out/${1:-hfd}; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -k "huffman or parity or fullsize or golden or default or secondary" > $O/tests.txt 2>&1
echo "tests exit $?" >> $O/tests.txt
timeout 600 python bench.py --no-cpu > $O/bench_c4.json 2> $O/bench_c4.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"hf_|huffman" -c 40 --csv --log-file $O/launches_c4.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-parity > /dev/null 2>&1
