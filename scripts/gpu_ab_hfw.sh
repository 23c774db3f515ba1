#!/bin/bash
# Huffman encode passes on dense (C1, a C5 field) and sparse (C4) streams + C5/C4 bench
O=gpurun_out/${1:-ab3}; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -x -q -k "huffman or hist or flag or fullsize" > $O/tests.txt 2>&1; echo "tests exit $?" >> $O/tests.txt
for c in "512x512x512 default 1e-3 c5f" "100x500x500 default 1e-4 c1" "280953867 default 1e-4 c4"; do set -- $c
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"hf_write2|hist_smem|hf_count" -c 3 --csv --log-file $O/l_$4.csv python scripts/prof_roundtrip.py $1 $2 $3 > /dev/null 2>&1
done
timeout 900 python bench.py --workload c5 --no-cpu --steps 5 > $O/bench_c5.json 2> $O/bench_c5.err
timeout 900 python bench.py --no-cpu > $O/bench_c4.json 2> $O/bench_c4.err
