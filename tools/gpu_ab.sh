cd /root/repo
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/ab_tests.log 2>&1
echo "rc=$?" >> gpurun_out/ab_tests.log
python tools/profile_solve.py 256 10 > gpurun_out/ab_prof.log 2>&1
MM_STENCIL_MARCH=0 python tools/profile_solve.py 256 10 >> gpurun_out/ab_prof.log 2>&1
