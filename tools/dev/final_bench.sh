python bench.py --steps 5 --warmup 3 > gpurun_out/r2_bench_final.json 2> gpurun_out/r2_bench_final.err
python bench.py --steps 3 --warmup 3 --solver cbshv --precision f16 --no-cpu > gpurun_out/r2_bench_cbshv16.json 2>> gpurun_out/r2_bench_final.err
python bench.py --steps 3 --warmup 3 --solver cbshv --no-cpu > gpurun_out/r2_bench_cbshv.json 2>> gpurun_out/r2_bench_final.err
python bench.py --steps 3 --warmup 3 --precision f16 --no-cpu > gpurun_out/r2_bench_ndb16.json 2>> gpurun_out/r2_bench_final.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r2_launches_final.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-parity --no-e2e > /dev/null 2>&1
