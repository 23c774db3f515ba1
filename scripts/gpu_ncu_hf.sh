O=gpurun_out/${1:-r02n}; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"hf_write2|hf_count|hf_write_dec2|lz1d_summary2|hist_smem|lz1d_fill2" -c 6 -o $O/c4_stream python scripts/prof_roundtrip.py 280953867 default 1e-4 > $O/ncu_c4s.log 2>&1
