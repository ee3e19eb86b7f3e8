timeout 600 python -m pytest tests -q -m gpu -x > gpurun_out/q_tests.log 2>&1
python tools/profile_iter.py 256 6 > gpurun_out/q_prof.log 2>&1
