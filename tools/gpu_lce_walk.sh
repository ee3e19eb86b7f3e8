# LCE point-walking kernel: parity tests, 64^3 counters (diagnostics build), 256^3 timing (normal build)
cd /root/repo
timeout 900 python -m pytest tests/test_gpu_lce.py tests/test_gpu_scenarios.py -q -x 2>&1 | tail -3
timeout 600 python tools/lce_perf.py 256 2000 3 2>&1 | tail -3
MM_NVCC_FLAGS="-DMM_LCE_STATS=1" python -c "from paper_2010_06697_b200 import build; build.build(force=True)" > /dev/null 2>&1
timeout 600 python tools/lce_perf.py 64 2000 3 | tail -10
