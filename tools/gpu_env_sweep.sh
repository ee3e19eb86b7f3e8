# runtime-knob sweep at the default bench: each argument is an env assignment list
cd /root/repo
for v in "$@"; do
  env $v timeout 600 python bench.py --no-cpu-baseline > gpurun_out/es.json 2>/dev/null
  python - "$v" <<'PY'
import json,sys
d=json.load(open('gpurun_out/es.json'))
st=d['stages']
print(sys.argv[1], 'ms/it %.3f'%d['ms_per_step'], {k:round(v['ms_per_launch'],3) for k,v in st.items() if v['launches']})
PY
done
