# side-buffered Clenshaw fp16 launches (DASH_SIDEBUF=1, default) vs the shared staging buffer (0)
for sb in 1 0; do echo "== DASH_SIDEBUF=$sb"; DASH_SIDEBUF=$sb timeout 300 python tools/solver_bench.py --solver cheb --n 1820 --b 1024 --mode f16 --reps 2 2>&1 | grep "cheb"; done
DASH_GEMM_DEBUG=2 timeout 300 python tools/solver_bench.py --solver cheb --n 1820 --b 1024 --mode f16 --reps 1 2>&1 | grep "\[gemm\]" | sort | uniq -c | sort -rn | head -2
timeout 300 python tools/solver_bench.py --n 1820 --b 1024 --mode f16 --reps 2 2>&1 | grep "ndb: total"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_parity.py tests/test_gpu_variants.py -q -x 2>&1 | tail -3
