# parity tests + default bench stage times
cd /root/repo
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scenarios.py -q -x > gpurun_out/q_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/q_pytest.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/q_bench.json 2>/dev/null
python - <<'PY'
import json
d=json.load(open('gpurun_out/q_bench.json'))
st=d['stages']
print('ms/it %.3f'%d['ms_per_step'], 'e2e %.3g'%d['e2e']['value'], {k:round(v['ms_per_launch'],3) for k,v in st.items() if v['launches']})
PY
