cd /root/repo
timeout 300 python tools/lce_perf.py 64 200 3 > gpurun_out/lce64.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_lce3d" -s 2 -c 1 \
    -o gpurun_out/lce3d python tools/lce_perf.py 64 200 3 > gpurun_out/lce_ncu.log 2>&1
echo done
