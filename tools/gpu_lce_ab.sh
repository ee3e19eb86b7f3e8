# A/B of mm_lce.cu build variants on the 3D polydomain LCE local step (128^3,
# max_local 200): local-stage time per variant, REPS rounds
cd /root/repo
for rep in $(seq 1 ${REPS:-2}); do
for v in "$@"; do
  touch paper_2010_06697_b200/csrc/mm_lce.cu
  MM_NVCC_FLAGS="$v" python -c "from paper_2010_06697_b200 import build; build.build()" > gpurun_out/ab_build.log 2>&1 || tail -3 gpurun_out/ab_build.log
  echo "[$v] $(timeout 600 python tools/lce_perf.py 128 200 3 2>/dev/null | tail -1)"
done
done
