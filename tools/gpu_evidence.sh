# round evidence: bench line (no profiler), launch list, one full capture per stage kernel,
# LCE config-3 timing
cd /root/repo
python bench.py > gpurun_out/ev_bench.json 2> gpurun_out/ev_bench.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ev_ref.json 2> gpurun_out/ev_ref.err
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ev_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev_launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ev_launch.log 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:"k_update_local|k_row_fwd|k_row_inv|k_col|k_res_march" -s 22 -c 8 \
    -o gpurun_out/ev_full python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ev_full.log 2>&1

echo done
