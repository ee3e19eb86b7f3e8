cd /root/repo
timeout 900 python -m pytest tests/test_gpu_slab.py tests/test_snapshot.py -q -x > gpurun_out/slab2.log 2>&1
echo "rc=$?" >> gpurun_out/slab2.log
