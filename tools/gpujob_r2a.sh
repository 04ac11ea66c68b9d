# Round-2 first look: host of the box, cfg5/cfg4 bench lines and one ncu --set full
# capture of the cfg5 dense eval and window-cluster hess_apply (after the bench exited 0).
set -x
mkdir -p gpurun_out/r2a
(free -g; nproc; lscpu | head -20; nvidia-smi) > gpurun_out/r2a/host.txt 2>&1
python -c "import paper_2603_07156_b200.build as b; b.build(verbose=True)" > gpurun_out/r2a/build.log 2>&1
timeout 900 python bench.py --config 5 --no-cpu --no-solve --steps 2 --warmup 3 > gpurun_out/r2a/bench_cfg5.json 2>gpurun_out/r2a/bench_cfg5.err; echo c5_exit=$?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"^k_(eval|hv_wc|sparsify|test_a|test_c)$" -c 5 -o gpurun_out/r2a/cfg5_full python bench.py --config 5 --no-cpu --no-solve --steps 1 --warmup 3 > gpurun_out/r2a/ncu5.log 2>&1; echo ncu5_exit=$?
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"^k_(eval|hv_wc)$" -c 2 -o gpurun_out/r2a/cfg4_full python bench.py --config 4 --no-cpu --no-solve --steps 1 --warmup 3 > gpurun_out/r2a/ncu4.log 2>&1; echo ncu4_exit=$?
# summaries on the box (the .ncu-rep files may exceed the copy-back limit)
for f in gpurun_out/r2a/*.ncu-rep; do
  ncu -i "$f" --page raw --csv > "${f%.ncu-rep}_raw.csv" 2>/dev/null
  ncu -i "$f" --page details --csv > "${f%.ncu-rep}_details.csv" 2>/dev/null
done
du -sh gpurun_out/r2a/*
tot=$(du -sm gpurun_out | cut -f1); if [ "$tot" -gt 60 ]; then rm -f gpurun_out/r2a/*.ncu-rep; fi
