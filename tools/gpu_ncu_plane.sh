cd /root/repo
export MM_PLANE_CS=4
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/np_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_plane" -s 2 -c 1 \
    -o gpurun_out/plane_full2 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/np_full.log 2>&1
echo rc=$?
