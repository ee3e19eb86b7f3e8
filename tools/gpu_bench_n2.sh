# the bench's N > 1 path (solve(comm=TorchComm): slab decomposition, push and
# collective transposes) with two ranks on one GPU (gloo: NCCL refuses two
# ranks per device; exchanges staged through the host)
cd /root/repo
for ex in push collective; do
MM_BENCH_DEVICE=0 MM_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --standalone --local-addr 127.0.0.1 \
    --nproc-per-node 2 bench.py --gpus 2 --grid ${N:-64} --steps 5 --warmup 3 --exchange $ex 2>&1 | grep -v Warning | tail -3
done
