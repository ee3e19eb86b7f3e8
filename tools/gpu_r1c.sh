# GPU tests + stage profile + a short bench line
cd /root/repo
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/c_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/c_tests.log
python tools/profile_solve.py 256 10 > gpurun_out/c_prof.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 5 --no-cpu-baseline > gpurun_out/c_bench.json 2> gpurun_out/c_bench.err
