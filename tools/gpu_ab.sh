# A/B of build variants at the default bench (K = 50): each argument is a set of
# nvcc flags applied to SRC (default mm_local.cu); REPS rounds (default 2);
# TESTS=1 also runs the GPU suite once on the last variant; BENCH_ARGS are
# passed to bench.py (e.g. "--grid 512 --steps 10 --warmup 3").
# e.g.  SRC=mm_project.cu bash tools/gpu_ab.sh "-DMM_PLANE_PPT=8" "-DMM_PLANE_PPT=16"
cd /root/repo
summ() {
python - "$1" <<'PY'
import json,sys
d=json.load(open('gpurun_out/ab.json'))
st=d['stages']
print(sys.argv[1], 'ms/it %.3f'%d['ms_per_step'], 'sweeps/vox %.3f'%d['roofline_local_fp64']['point_sweeps_per_voxel_iter'], {k:round(v['ms_per_launch'],3) for k,v in st.items() if v['launches']})
PY
}
for rep in $(seq 1 ${REPS:-2}); do
for v in "$@"; do
  touch paper_2010_06697_b200/csrc/${SRC:-mm_local.cu}
  MM_NVCC_FLAGS="$v" python -c "from paper_2010_06697_b200 import build; build.build()" > gpurun_out/ab_build.log 2>&1 || tail -3 gpurun_out/ab_build.log
  timeout 600 python bench.py --no-cpu-baseline $BENCH_ARGS > gpurun_out/ab.json 2>/dev/null; summ "[$v]"
done
done
if [ -n "$TESTS" ]; then
  timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/ab_pytest.log 2>&1; echo "pytest [$v] rc=$?"; tail -2 gpurun_out/ab_pytest.log
fi
