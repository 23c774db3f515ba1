#!/bin/bash
# 2D shared-memory-tiled G-Interp: parity (GPU suite) + C3 A/B against the per-pass kernels.
O=gpurun_out/${1:-i2d}
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q ${TESTK:+-k "$TESTK"} > $O/tests.txt 2>&1
echo "tests exit $?" >> $O/tests.txt
timeout 300 python bench.py --workload c3 --no-cpu > $O/bench_c3.json 2> $O/bench_c3.err
FZB_INTERP_PASSES=1 timeout 300 python bench.py --workload c3 --no-cpu > $O/bench_c3_passes.json 2> $O/bench_c3_passes.err
timeout 300 python bench.py --workload c3 --no-cpu --pipeline quality > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c3.csv python bench.py --workload c3 --steps 2 --warmup 1 --no-cpu --no-parity > /dev/null 2>&1
