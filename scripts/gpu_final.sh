#!/bin/bash
# Round-end GPU session: parity suite, smoke, every bench workload + the
# reference arm, ncu launch lists and --set full captures (CSV on the box).
# Usage (via gpurun): bash scripts/gpu_final.sh TAG
TAG=${1:-r02final}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err
for w in c1 c2 c3 c5; do timeout 900 python bench.py --workload $w --no-cpu > $O/bench_$w.json 2> $O/bench_$w.err; done
for p in dq-speed dq-default; do timeout 600 python bench.py --workload c2 --pipeline $p --no-cpu > $O/bench_c2_$p.json 2> $O/bench_c2_$p.err; done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref_c4.json 2> $O/bench_ref_c4.err
bash scripts/gpu_launches.sh $TAG
bash scripts/gpu_profiles.sh $TAG
echo done > $O/done.txt
