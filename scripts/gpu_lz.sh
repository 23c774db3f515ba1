#!/bin/bash
# Lorenzo A/B + parity + bench (ad-hoc GPU session)
O=gpurun_out/${1:-lz}
mkdir -p $O
timeout 180 python scripts/lz_micro.py ${LZ_SHAPES} > $O/lz_micro.txt 2>&1; echo "rc=$?" >> $O/lz_micro.txt
if grep -q "codes_eq': True" $O/lz_micro.txt; then
  timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
  timeout 300 python bench.py --no-cpu > $O/bench_c2.json 2> $O/bench_c2.err
  timeout 300 python bench.py --workload c1 --no-cpu > $O/bench_c1.json 2> $O/bench_c1.err
  timeout 300 python scripts/prof_e2e.py > $O/e2e_c2.txt 2>&1
fi
