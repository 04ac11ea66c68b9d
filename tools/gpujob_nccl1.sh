# NCCL binding on one GPU: the one-rank self-test (pytest) and bench.py under torchrun with one rank
set -x
T=${1:-nccl1}
mkdir -p gpurun_out/$T
timeout 900 python -m pytest tests/test_gpu_multirank.py -m gpu -q -x -k nccl > gpurun_out/$T/pytest_nccl.log 2>&1; echo nccl_exit=$?; tail -15 gpurun_out/$T/pytest_nccl.log
OTB_NCCL_SELFTEST=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29711 bench.py --gpus 1 --config 4 --steps 3 --warmup 3 --no-cpu --secondary "" --e2e-steps 1 > gpurun_out/$T/bench4_nccl.json 2>gpurun_out/$T/bench4_nccl.err; echo b4_exit=$?; tail -5 gpurun_out/$T/bench4_nccl.err
OTB_NCCL_SELFTEST=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29712 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu --secondary "" --e2e-steps 1 > gpurun_out/$T/bench5_nccl.json 2>gpurun_out/$T/bench5_nccl.err; echo b5_exit=$?; tail -5 gpurun_out/$T/bench5_nccl.err
python tools/bench_brief.py gpurun_out/$T/bench4_nccl.json gpurun_out/$T/bench5_nccl.json
