cd /root/repo
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/ab3_tests.log 2>&1
echo "rc=$?" >> gpurun_out/ab3_tests.log
for i in 1 2; do
MM_T_FIELD=0 python tools/profile_solve.py 256 20 >> gpurun_out/ab3_prof.log 2>&1
MM_T_FIELD=1 python tools/profile_solve.py 256 20 >> gpurun_out/ab3_prof.log 2>&1
done
