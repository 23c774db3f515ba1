#!/bin/bash
# One GPU session: parity tests, smoke, bench (all workloads + reference arm),
# ncu launch lists + full captures of the top kernels.
# Usage (via gpurun): bash scripts/gpu_round.sh TAG [quick]
TAG=${1:-r01}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
for w in c1 c3 c4 c5; do timeout 600 python bench.py --workload $w --no-cpu > $O/bench_$w.json 2> $O/bench_$w.err; done
timeout 600 python bench.py --workload c5d --no-cpu > $O/bench_c5d.json 2> $O/bench_c5d.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref_c2.json 2> $O/bench_ref_c2.err
if [ "$2" != "quick" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c2.csv python bench.py --steps 2 --warmup 1 --no-cpu > $O/ncu_launch.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c1.csv python scripts/prof_roundtrip.py 100x500x500 default 1e-4 > $O/ncu_launch_c1.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c3.csv python scripts/prof_roundtrip.py 1800x3600 quality 1e-4 > $O/ncu_launch_c3.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c4.csv python scripts/prof_roundtrip.py 280953867 default 1e-4 > $O/ncu_launch_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"lz7_kernel|bs_enc4|bs_dec3" -c 4 -o $O/c2_full python scripts/prof_roundtrip.py 512x512x512 speed 1e-3 > $O/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"hf_|huffman_build|hist_" -c 9 -o $O/c1_full python scripts/prof_roundtrip.py 100x500x500 default 1e-4 > $O/ncu_full_c1.log 2>&1
fi
echo done
