# ncu source-level capture of the 1D walker (C4)
O=gpurun_out/r02f; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"lz1d_walk3" -c 1 -o $O/walk3 python scripts/prof_roundtrip.py 280953867 default 1e-4 > $O/ncu_walk3.log 2>&1
