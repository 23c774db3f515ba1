# ncu --set full of kernels matching $2 in a C4 round trip
O=gpurun_out/${1}; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$2" -c ${3:-1} -o $O/k python scripts/prof_roundtrip.py ${4:-280953867} ${5:-default} ${6:-1e-4} > $O/ncu.log 2>&1
