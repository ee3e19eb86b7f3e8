# full ncu captures (source counters) of the fused K2 and the plane pass at a
# steady-state 256^3 iteration, for the source-level hot-spot read-out
cd /root/repo
python bench.py --steps 3 --warmup 10 --no-cpu-baseline > gpurun_out/hot_plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_update_local<.int.0, .int.9, .int.0, .bool.1>|k_plane" -s 20 -c 2 \
    -o gpurun_out/hot_full python bench.py --steps 3 --warmup 10 --no-cpu-baseline > gpurun_out/hot_full.log 2>&1
echo rc=$?
