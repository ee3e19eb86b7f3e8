# fused K2 block shape variants (MM_LOCAL_THREADS x LOCAL_MIN_BLOCKS, same 128-register budget)
cd /root/repo
for v in "128 4" "64 8" "32 16"; do
  set -- $v
  MM_NVCC_FLAGS="-DMM_LOCAL_THREADS=$1 -DLOCAL_MIN_BLOCKS=$2" python -c "from paper_2010_06697_b200 import build; build.build(force=True)" > gpurun_out/k2b.log 2>&1 || tail -3 gpurun_out/k2b.log
  timeout 600 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/k2v.json 2>/dev/null
  python - "$v" <<'PY'
import json,sys
d=json.load(open('gpurun_out/k2v.json'))
st=d['stages']
print('threads,minb', sys.argv[1], 'ms/it %.3f'%d['ms_per_step'], {k:round(v['ms_per_launch'],3) for k,v in st.items() if v['launches']})
PY
done
