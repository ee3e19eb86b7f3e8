# plane pass: DRAM traffic and time per cluster size (one capture each)
cd /root/repo
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/np_plain.log 2>&1
for cs in 4 8 16; do
  MM_PLANE_CS=$cs ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_plane" -s 2 -c 1 --csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | grep -E "k_plane" | awk -F'","' -v cs=$cs '{print "CS=" cs, $(NF-2), $(NF-1), $NF}'
done
