cd /root/repo
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/f_tests.log 2>&1
echo "rc=$?" >> gpurun_out/f_tests.log
python tools/e2e_profile.py 256 10 > gpurun_out/e2e_prof.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err
