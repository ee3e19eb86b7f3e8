cd /root/repo
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/e_tests.log 2>&1
echo "rc=$?" >> gpurun_out/e_tests.log
python tools/e2e_profile.py 256 10 > gpurun_out/e2e_prof.log 2>&1
