python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncl_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_descent|k_row_inv|k_col" -s 9 -c 5 \
    -o gpurun_out/local_r1b python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncl.log 2>&1
echo done
