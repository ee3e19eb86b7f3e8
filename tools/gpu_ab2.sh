cd /root/repo
for i in 1 2; do
MM_STENCIL_MARCH=0 python tools/profile_solve.py 256 20 >> gpurun_out/ab2_prof.log 2>&1
MM_STENCIL_MARCH=1 python tools/profile_solve.py 256 20 >> gpurun_out/ab2_prof.log 2>&1
done
