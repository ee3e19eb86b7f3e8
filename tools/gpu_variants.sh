cd /root/repo
for v in variants_tmp/*.so; do
  cp $v paper_2010_06697_b200/lib/libmm_admm.so
  echo "== $v" >> gpurun_out/var.log
  python tools/profile_solve.py 256 20 >> gpurun_out/var.log 2>&1
done
