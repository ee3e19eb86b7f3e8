# LCE 3D work counters (diagnostics build) at 64^3 polydomain, one outer iteration
cd /root/repo
MM_NVCC_FLAGS="-DMM_LCE_STATS=1" python -c "from paper_2010_06697_b200 import build; build.build(force=True)" > /dev/null 2>&1
timeout 600 python tools/lce_perf.py 64 2000 3
