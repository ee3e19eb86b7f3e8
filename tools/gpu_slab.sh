timeout 600 python -m pytest tests/test_gpu_slab.py -q -x > gpurun_out/s_tests.log 2>&1
timeout 600 python -m pytest tests -q -m gpu > gpurun_out/s_all.log 2>&1
python tools/profile_solve.py 256 10 > gpurun_out/s_prof.log 2>&1
