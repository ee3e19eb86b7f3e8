cd /root/repo
timeout 600 python -m pytest tests/test_gpu_lce.py -q -x > gpurun_out/lce_t.log 2>&1
echo "rc=$?" >> gpurun_out/lce_t.log
timeout 300 python tools/lce_perf.py 64 200 3 > gpurun_out/lce64.log 2>&1
