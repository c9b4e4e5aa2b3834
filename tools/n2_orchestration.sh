# bench.py's N>1 path (torchrun, transport selection, exchange report, e2e) exercised on
# a single-GPU box: two ranks on GPU 0, gloo host-staged exchanges, NCCL transport
# forced (the P2P transport would make two kernels on one GPU wait on each other).
# Not a benchmark: the numbers are meaningless, rc and the JSON keys are the point.
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29611 bench.py --gpus 2 --dist-backend gloo --same-device --transport nccl \
    --steps 3 --warmup 3 --e2e-steps 1 > gpurun_out/n2.json 2> gpurun_out/n2.err; echo "cgbn arm rc=$?"
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29612 bench.py --impl reference --gpus 2 --steps 3 --warmup 3 \
    > gpurun_out/n2ref.json 2> gpurun_out/n2ref.err; echo "reference arm rc=$?"
