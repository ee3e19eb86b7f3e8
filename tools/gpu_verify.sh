# re-entry check: GPU test suite, smoke, default bench line
cd /root/repo
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/v_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/v_pytest.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/v_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/v_bench.json 2> gpurun_out/v_bench.err; echo "bench rc=$?"
cat gpurun_out/v_bench.json | cut -c1-400
