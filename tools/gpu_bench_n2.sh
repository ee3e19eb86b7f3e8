# the bench's N > 1 path (slab decomposition, push exchange over CUDA IPC) with two ranks on one GPU
cd /root/repo
MM_BENCH_DEVICE=0 MM_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --standalone --local-addr 127.0.0.1 \
    --nproc-per-node 2 bench.py --gpus 2 --steps 5 --warmup 3 2>&1 | grep -v Warning | tail -5
