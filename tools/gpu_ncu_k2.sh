cd /root/repo
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/k2_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_update_local" -s 2 -c 1 \
    -o gpurun_out/k2_full python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/k2_full.log 2>&1
echo rc=$?
