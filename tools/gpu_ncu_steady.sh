cd /root/repo
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ns_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on \
    -k regex:"k_update_local|k_row_fwd|k_row_inv|k_col|k_grad" -s 22 -c 8 \
    -o gpurun_out/steady python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ns.log 2>&1
echo done
