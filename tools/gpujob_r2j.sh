set -x
mkdir -p gpurun_out/r2j
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "dense_rho or eval_post or pcg" > gpurun_out/r2j/pytest.log 2>&1; echo t_exit=$?; tail -3 gpurun_out/r2j/pytest.log
timeout 900 python bench.py --no-cpu --no-solve --e2e-steps 0 --secondary "" --steps 3 > gpurun_out/r2j/bench5.json 2>gpurun_out/r2j/bench5.err; echo b5_exit=$?
OTB_LIB=$PWD/paper_2603_07156_b200/libotb_norr.so timeout 900 python bench.py --no-cpu --no-solve --e2e-steps 0 --secondary "" --steps 3 > gpurun_out/r2j/bench5_norr.json 2>gpurun_out/r2j/bench5_norr.err; echo b5n_exit=$?
