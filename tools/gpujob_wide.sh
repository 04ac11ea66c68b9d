# WIDE (1024-thread) self-fed dense passes: per-kind mask sweep at config 5 (and 4)
# kinds: eval 1, test_a 4, test_b 8, test_c 16, test_c+metrics 32, sparsify_dense 512
T=${1:-wide}
mkdir -p gpurun_out/$T
for cfg in 5 4; do
for w in 0 573 525 1 4 8 48 512; do
  OTB_DENSE_WIDE=$w OTB_LIB=$PWD/_exp/main/libotb.so timeout 600 python bench.py --config $cfg --no-cpu --no-solve --e2e-steps 0 --secondary "" --steps 3 > gpurun_out/$T/c${cfg}_w$w.json 2>gpurun_out/$T/c${cfg}_w$w.err || tail -3 gpurun_out/$T/c${cfg}_w$w.err
  echo "cfg$cfg wide=$w"; python tools/bench_brief.py gpurun_out/$T/c${cfg}_w$w.json
done; done
