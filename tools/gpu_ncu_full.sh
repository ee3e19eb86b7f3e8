# one full ncu capture per stage kernel at a steady-state fused iteration (launch order per
# iteration: K2, A, plane, E [speculative front], K1; 15 matching launches in the warm-up solve)
cd /root/repo
python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/ev_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on \
    -k regex:"k_update_local|k_row_fwd|k_row_inv|k_plane|k_res_march" -s 24 -c 5 \
    -o gpurun_out/ev_full python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/ev_full.log 2>&1
echo rc=$?
