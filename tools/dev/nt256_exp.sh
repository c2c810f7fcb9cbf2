# NT = 256 ring experiment: split launches on 256-wide pair tiles (DASH_NT=2562), K-block 32 / 64
python tools/solver_bench.py --n 1820 --b 1024 --mode f32 --reps 2 2>&1 | grep "ndb:"
DASH_NT=2562 DASH_KB=32 python tools/solver_bench.py --n 1820 --b 1024 --mode f32 --reps 2 2>&1 | grep "ndb:"
DASH_NT=2562 DASH_KB=64 python tools/solver_bench.py --n 1820 --b 1024 --mode f32 --reps 2 2>&1 | grep "ndb:"
DASH_NT=2562 DASH_KB=32 DASH_GEMM_DEBUG=2 python tools/solver_bench.py --n 1820 --b 1024 --mode f32 --reps 1 2>&1 | grep "\[gemm\]" | sort | uniq -c | sort -rn | head -3
DASH_GEMM_DEBUG=2 python tools/solver_bench.py --n 1820 --b 1024 --mode f32 --reps 1 2>&1 | grep "\[gemm\]" | sort | uniq -c | sort -rn | head -3
DASH_NT=2562 DASH_KB=32 timeout 300 python tools/floor_probe.py --kmax 12 2>&1 | head -12
DASH_NT=2562 DASH_KB=32 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_parity.py -q -x 2>&1 | tail -3
