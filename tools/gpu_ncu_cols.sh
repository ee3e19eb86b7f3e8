python bench.py --n 256 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/nc_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_colp|k_row" -s 8 -c 4 \
    -o gpurun_out/cols_r1c python bench.py --n 256 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/nc.log 2>&1
echo done
