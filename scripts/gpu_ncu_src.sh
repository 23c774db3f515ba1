# ncu --set full of one kernel (regex $2) in a round trip; source page + raw exported on the box
O=gpurun_out/${1}; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$2" -c ${3:-1} -o /tmp/k python scripts/prof_roundtrip.py ${4:-280953867} ${5:-default} ${6:-1e-4} > $O/ncu.log 2>&1
ncu -i /tmp/k.ncu-rep --page source --csv --print-source sass > $O/src.csv 2>/dev/null
ncu -i /tmp/k.ncu-rep --page raw --csv > $O/raw.csv 2>/dev/null
rm -f /tmp/k.ncu-rep
