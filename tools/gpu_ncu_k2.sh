# full capture of the fused K2 kernel at a steady-state iteration (the 11th launch)
cd /root/repo
python bench.py --steps 3 --warmup 10 --no-cpu-baseline > gpurun_out/k2_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_update_local" -s 10 -c 1 \
    -o gpurun_out/k2_full python bench.py --steps 3 --warmup 10 --no-cpu-baseline > gpurun_out/k2_full.log 2>&1
echo rc=$?
