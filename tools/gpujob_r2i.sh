set -x
mkdir -p gpurun_out/r2i
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "dense_rho or hess_apply or cluster_paths or step_pipeline or pcg" > gpurun_out/r2i/pytest_hv.log 2>&1; echo hv_exit=$?; tail -3 gpurun_out/r2i/pytest_hv.log
timeout 300 ./tools/tma_bench > gpurun_out/r2i/tma_bench.txt 2>&1; echo tma_exit=$?
timeout 900 python bench.py --no-cpu --no-solve --e2e-steps 0 --secondary "2,3" --steps 3 > gpurun_out/r2i/bench5.json 2>gpurun_out/r2i/bench5.err; echo b5_exit=$?
OTB_DENSE_CL=6 timeout 900 python bench.py --no-cpu --no-solve --e2e-steps 0 --secondary "" --steps 3 > gpurun_out/r2i/bench5_cl6.json 2>gpurun_out/r2i/bench5_cl6.err; echo b5cl6_exit=$?
OTB_LIB=$PWD/paper_2603_07156_b200/libotb_t512.so OTB_DENSE_CL=6 OTB_DENSE_NT=480 timeout 900 python bench.py --no-cpu --no-solve --e2e-steps 0 --secondary "2,3" --steps 3 > gpurun_out/r2i/bench5_t512.json 2>gpurun_out/r2i/bench5_t512.err; echo b5t512_exit=$?
