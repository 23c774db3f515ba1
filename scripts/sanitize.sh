#!/bin/bash
# compute-sanitizer sweeps over small GPU parity cases (memcheck: every
# kernel family; racecheck / synccheck: the v7 wavefront's shared-memory
# rings on one small shape).  Usage (via gpurun): bash scripts/sanitize.sh TAG
O=gpurun_out/${1:-san}
mkdir -p $O
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_kernels.py -x -q \
  -k "v7_lorenzo_shapes or bitshuffle_sizes or huffman_alphabets or batch or quality_device or nonfinite or 2d" \
  > $O/memcheck_kernels.txt 2>&1
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -x -q \
  -k "cuda_graph or wire or c4 or interp" > $O/memcheck_parity.txt 2>&1
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python scripts/lz_micro.py 9x33x64 > $O/racecheck_lz.txt 2>&1
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python scripts/lz_micro.py 9x33x64 > $O/synccheck_lz.txt 2>&1
for f in $O/*.txt; do echo "$f: $(grep -h 'ERROR SUMMARY' $f | tail -1)"; done
