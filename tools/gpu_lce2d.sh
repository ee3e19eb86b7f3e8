# 2D LCE: parity tests and a 512^2 polydomain timing
cd /root/repo
timeout 900 python -m pytest tests/test_gpu_lce.py tests/test_gpu_scenarios.py -q -x 2>&1 | tail -2
timeout 600 python tools/lce_perf.py 512 2000 2 2>&1 | tail -3
