timeout 600 python -m pytest tests -q -m gpu -x > gpurun_out/f_tests.log 2>&1
python tools/profile_solve.py 256 10 > gpurun_out/f_prof.log 2>&1
MM_FUSE=0 python tools/profile_solve.py 256 10 >> gpurun_out/f_prof.log 2>&1
