#!/bin/bash
# One GPU session: parity tests, smoke, bench (all workloads), ncu launch list + full capture.
# Usage (via gpurun): bash scripts/gpu_round.sh TAG [quick]
TAG=${1:-r01}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
for w in c1 c3 c4; do timeout 600 python bench.py --workload $w --no-cpu > $O/bench_$w.json 2> $O/bench_$w.err; done
if [ "$2" != "quick" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c2.csv python bench.py --steps 2 --warmup 1 --no-cpu > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lz_wave4_kernel -c 2 -o $O/lz_full python scripts/prof_roundtrip.py 512x512x512 speed 1e-3 > $O/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bs_ -c 3 -o $O/bs_full python scripts/prof_roundtrip.py 512x512x512 speed 1e-3 > $O/ncu_bs.log 2>&1
fi
echo done
