# ncu launch lists (per-kernel durations) of one round trip per config
O=gpurun_out/${1:-r02k}; mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c4.csv python scripts/prof_roundtrip.py 280953867 default 1e-4 > $O/ncu_c4.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c2.csv python scripts/prof_roundtrip.py 512x512x512 speed 1e-3 > $O/ncu_c2.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c1.csv python scripts/prof_roundtrip.py 100x500x500 default 1e-4 > $O/ncu_c1.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c3.csv python scripts/prof_roundtrip.py 1800x3600 quality 1e-4 > $O/ncu_c3.log 2>&1
