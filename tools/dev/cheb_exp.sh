# Chebyshev fp16 epilogue cost breakdown: DASH_EXP knobs (timing only; results invalid with knobs != 0)
for x in 0 2 4 8 12 256 260; do echo "== DASH_EXP=$x"; DASH_EXP=$x python tools/solver_bench.py --solver cheb --n 1820 --b 1024 --mode f16 --reps 1 2>&1 | grep "cheb:" | head -1; done
DASH_GEMM_DEBUG=2 python tools/solver_bench.py --solver cheb --n 1820 --b 1024 --mode f16 --reps 1 2>&1 | grep "\[gemm\]" | sort | uniq -c | sort -rn | head -2
