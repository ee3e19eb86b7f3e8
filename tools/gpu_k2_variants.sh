# fused K2 register budget variants (LOCAL_MIN_BLOCKS): rebuild mm_local per variant, bench stage times
cd /root/repo
for v in 3 4 5 6; do
  MM_NVCC_FLAGS="-DLOCAL_MIN_BLOCKS=$v" python -c "from paper_2010_06697_b200 import build; build.build(force=True)" > /dev/null 2>&1
  timeout 600 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/k2v.json 2>/dev/null
  python - "$v" <<'PY'
import json,sys
d=json.load(open('gpurun_out/k2v.json'))
st=d['stages']
print('MINB', sys.argv[1], 'ms/it %.3f'%d['ms_per_step'], {k:round(v['ms_per_launch'],3) for k,v in st.items() if v['launches']})
PY
done
