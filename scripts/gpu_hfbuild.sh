#!/bin/bash
# Huffman build: large-alphabet parity tests + build micro-benchmark (+ phase cycles)
O=gpurun_out/${1:-hfb}; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -x -q -k "huffman or codebook" > $O/tests.txt 2>&1
timeout 300 python scripts/hf_build_micro.py > $O/micro.txt 2>&1
FZB_SO=paper_2509_20563_b200/_build/var/libfzb200_tim.so timeout 300 python scripts/hf_build_micro.py > $O/micro_tim.txt 2>&1
