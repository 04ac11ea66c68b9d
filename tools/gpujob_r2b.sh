# Round 2: multi-rank local group, dense drop-ins, config seeds / full-size
# properties, then the whole GPU suite; cluster packing probe.
set -x
mkdir -p gpurun_out/r2b
./tools/cluster_probe > gpurun_out/r2b/cluster_probe.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_dropins.py -x -q > gpurun_out/r2b/pytest_new.log 2>&1; echo new_exit=$?; tail -15 gpurun_out/r2b/pytest_new.log
timeout 1500 python -m pytest tests/test_gpu_configs.py -q > gpurun_out/r2b/pytest_cfg.log 2>&1; echo cfg_exit=$?; tail -15 gpurun_out/r2b/pytest_cfg.log
timeout 1500 python -m pytest tests -m gpu -q --deselect tests/test_gpu_configs.py > gpurun_out/r2b/pytest_all.log 2>&1; echo all_exit=$?; tail -15 gpurun_out/r2b/pytest_all.log
