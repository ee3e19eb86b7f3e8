# speculative projection front: per-iteration time with and without, three grid sizes
cd /root/repo
for n in 64 128 256; do for s in 0 1; do
  MM_SPECULATE=$s timeout 600 python bench.py --grid $n --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/sp.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/sp.json')); print('n=$n spec=$s', round(d['ms_per_step'],4), '%.3g' % d['value'])"
done; done
