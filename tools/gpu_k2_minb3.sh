cd /root/repo
MM_NVCC_FLAGS="-DLOCAL_MIN_BLOCKS=3" python -c "from paper_2010_06697_b200 import build; build.build(force=True)" > gpurun_out/k2b.log 2>&1; echo build rc=$?; tail -2 gpurun_out/k2b.log
timeout 600 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/k2v.json 2> gpurun_out/k2v.err; echo bench rc=$?; tail -3 gpurun_out/k2v.err
python -c "
import json; d=json.load(open('gpurun_out/k2v.json')); print(d['ms_per_step'], {k:round(v['ms_per_launch'],3) for k,v in d['stages'].items() if v['launches']})"
