timeout 900 python -m pytest tests -q -m gpu > gpurun_out/lce_tests.log 2>&1
timeout 300 python tools/lce_perf.py 64 2000 3 > gpurun_out/lce_perf.log 2>&1
timeout 300 python tools/lce_perf.py 256 2000 2 >> gpurun_out/lce_perf.log 2>&1
