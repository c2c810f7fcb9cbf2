cd $GRAFT_REPO_ROOT
timeout 900 python bench.py > gpurun_out/bench_up.json 2> gpurun_out/bench_up.err
tail -1 gpurun_out/bench_up.json | cut -c1-300
timeout 600 python bench.py --precision f16 --no-cpu --steps 5 --warmup 3 > gpurun_out/bench_up_f16.json 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_up.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_list.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dash_gemm2 --launch-skip 24 --launch-count 1 -o gpurun_out/r1_gemm_up_yz python tools/solver_bench.py --n 1820 --b 1024 --iters 10 --mode f32 --reps 1 > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
