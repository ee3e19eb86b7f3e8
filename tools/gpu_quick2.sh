timeout 600 python -m pytest tests -q -m gpu -x > gpurun_out/q_tests.log 2>&1
MM_IMPLICIT_GRAD=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_lce.py -q -x > gpurun_out/q_tests_impl.log 2>&1
python tools/profile_iter.py 256 6 > gpurun_out/q_prof.log 2>&1
MM_IMPLICIT_GRAD=1 python tools/profile_iter.py 256 6 > gpurun_out/q_prof_impl.log 2>&1
