# N > 1 bench code paths on a single GPU: 2 ranks sharing GPU 0 with gloo collectives
O=gpurun_out/${1:-r02mr}; mkdir -p $O
FZB_BENCH_BACKEND=gloo timeout 900 python bench.py --gpus 2 --workload c5 --steps 2 --warmup 1 --no-parity > $O/c5_2ranks.json 2> $O/c5_2ranks.err
FZB_BENCH_BACKEND=gloo timeout 900 python bench.py --gpus 2 --steps 3 --warmup 1 --no-parity > $O/c4_2ranks.json 2> $O/c4_2ranks.err
