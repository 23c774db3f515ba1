mkdir -p gpurun_out/r02e
export FZB_SO=paper_2509_20563_b200/_build/var/libfzb200_timing.so
echo "spec" >> gpurun_out/r02e/walk.txt; timeout 300 python scripts/walk_timing.py >> gpurun_out/r02e/walk.txt 2>&1
echo "spec twice" >> gpurun_out/r02e/walk.txt; FZB_WALK_TWICE=1 timeout 300 python scripts/walk_timing.py >> gpurun_out/r02e/walk.txt 2>&1
echo "spec 1e-3" >> gpurun_out/r02e/walk.txt; timeout 300 python scripts/walk_timing.py 280953867 1e-3 >> gpurun_out/r02e/walk.txt 2>&1
unset FZB_SO
timeout 900 python -m pytest tests -m gpu -q -x -k "1d or c4 or C4 or particle or ws_reuse or zero or lorenzo or smooth1d" > gpurun_out/r02e/pytest.log 2>&1
timeout 600 python bench.py --no-cpu --no-parity > gpurun_out/r02e/bench_c4.json 2> gpurun_out/r02e/bench_c4.err
