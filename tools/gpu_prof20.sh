cd /root/repo
python tools/profile_solve.py 256 20 > gpurun_out/p20.log 2>&1
python tools/profile_solve.py 256 20 >> gpurun_out/p20.log 2>&1
