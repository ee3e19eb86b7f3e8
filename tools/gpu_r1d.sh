cd /root/repo
timeout 600 python -m pytest tests/test_gpu_scenarios.py -q -x > gpurun_out/d_scen.log 2>&1
echo "rc=$?" >> gpurun_out/d_scen.log
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/d_tests.log 2>&1
echo "rc=$?" >> gpurun_out/d_tests.log
