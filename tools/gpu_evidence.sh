# round evidence: bench line at the driver's K / W (no profiler), the LCE workload,
# the reference arm, launch list, one full capture per stage kernel, a 512^3 line
cd /root/repo
python bench.py --steps 20 --warmup 5 > gpurun_out/ev_bench.json 2> gpurun_out/ev_bench.err
python bench.py --workload lce --steps 2 --warmup 3 > gpurun_out/ev_lce.json 2> gpurun_out/ev_lce.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ev_ref.json 2> gpurun_out/ev_ref.err
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ev_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev_launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ev_launch.log 2>&1
bash tools/gpu_ncu_full.sh  # one full capture per stage kernel, steady state
timeout 900 python bench.py --grid 512 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ev_bench512.json 2> gpurun_out/ev_bench512.err
echo done
