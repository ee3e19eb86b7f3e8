# one full ncu capture of each k_lce3d mode launched in a split (Newton-compacted)
# local step: 128^3 polydomain, max_local 200 (large enough for the split schedule)
cd /root/repo
timeout 600 python tools/lce_perf.py 128 200 3 > gpurun_out/lce128.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_lce3d" -s 1 -c 3 \
    -o gpurun_out/lce3d python tools/lce_perf.py 128 200 3 > gpurun_out/lce_ncu.log 2>&1
echo rc=$?
