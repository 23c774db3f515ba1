#!/bin/bash
# Ad-hoc GPU session: micro latencies + e2e profile.
O=gpurun_out/${1:-q}
mkdir -p $O
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -fmad=false -o /tmp/lat scripts/micro/lat.cu && /tmp/lat > $O/lat.txt 2>&1
timeout 300 python scripts/prof_e2e.py > $O/e2e_c2.txt 2>&1
timeout 300 python scripts/prof_e2e.py 100x500x500 default 1e-4 > $O/e2e_c1.txt 2>&1
