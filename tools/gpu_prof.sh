# profile breakdown + bench + ncu on the top kernels (128^3 case)
python tools/profile_iter.py 256 6 > gpurun_out/prof3.log 2>&1
python bench.py --steps 10 --warmup 5 --no-cpu-baseline > gpurun_out/bench3.log 2>&1
python bench.py --n 128 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_descent|k_row_fwd|k_grad|k_col|k_row_inv" -s 20 -c 6 \
    -o gpurun_out/prof3 python bench.py --n 128 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu3.log 2>&1
echo done
