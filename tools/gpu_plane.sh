# plane-FFT check: bitwise equality with the row layout, parity tests, stage timing per cluster size
cd /root/repo
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pl_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pl_pytest.log
for v in "MM_PLANE_TK=8" "MM_PLANE_TK=4" "MM_PLANE_TK=4 MM_PLANE_CS=16" "MM_PLANE_TK=16 MM_PLANE_CS=4"; do
  env $v timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/pl_bench.json 2>/dev/null
  python - "$v" <<'PY'
import json,sys
d=json.load(open('gpurun_out/pl_bench.json'))
st=d['stages']
print(sys.argv[1], 'ms/it %.3f'%d['ms_per_step'], {k:round(v['ms_per_launch'],3) for k,v in st.items() if v['launches']})
PY
done
