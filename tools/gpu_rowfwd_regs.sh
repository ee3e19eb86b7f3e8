cd /root/repo
for r in 96 80; do
  MM_NVCC_FLAGS="-DMM_ROWFWD_REGS=$r" python -c "from paper_2010_06697_b200 import build; build.build(force=True)" > gpurun_out/rb.log 2>&1
  timeout 600 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/rv.json 2>/dev/null
  python -c "
import json,sys; d=json.load(open('gpurun_out/rv.json')); print('regs $r', d['ms_per_step'], {k:round(v['ms_per_launch'],3) for k,v in d['stages'].items() if v['launches']})"
done
