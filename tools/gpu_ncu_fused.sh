python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/nf_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_update_local" -s 0 -c 1 \
    -o gpurun_out/fused_r1b python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/nf.log 2>&1
echo done
