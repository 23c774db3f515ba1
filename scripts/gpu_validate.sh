#!/bin/bash
# Validation of the committed state: GPU suite, smoke, C4 + C2 bench, C2 ncu --set full (CSV)
O=gpurun_out/${1:-val}; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err
timeout 900 python bench.py --workload c2 --no-cpu > $O/bench_c2.json 2> $O/bench_c2.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c2.csv python scripts/prof_roundtrip.py 512x512x512 speed 1e-3 > /dev/null 2>&1
K='regex:^(?!at::|elementwise|vectorized|unrolled|distribution).*'
timeout 1200 ncu --set full --clock-control none --import-source on -k "$K" -c 40 -o /tmp/c2 python scripts/prof_roundtrip.py 512x512x512 speed 1e-3 > $O/ncu_c2.log 2>&1
ncu -i /tmp/c2.ncu-rep --page raw --csv > $O/raw_c2.csv 2>/dev/null; rm -f /tmp/c2.ncu-rep
