# LCE kernels: parity tests and the config-3 timing (256^3 polydomain, one outer iteration)
cd /root/repo
timeout 900 python -m pytest tests/test_gpu_lce.py tests/test_gpu_scenarios.py -q -x 2>&1 | tail -3
timeout 900 python tools/lce_perf.py 256 2000 3 2>&1 | tail -3
