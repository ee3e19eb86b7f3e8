# round-1 evidence: bench line, launch list and a full ncu capture of each stage kernel (256^3)
python bench.py --steps 10 --warmup 5 > gpurun_out/bench_r1.log 2>&1
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_plain_r1.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_r1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_descent|k_row_fwd|k_row_inv|k_col|k_grad" -s 21 -c 7 \
    -o gpurun_out/full_r1 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_r1.log 2>&1
echo done
