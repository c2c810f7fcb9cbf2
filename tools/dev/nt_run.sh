cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py -x -q 2>&1 | tail -2
run() { env "$@" DASH_GEMM_DEBUG=2 timeout 300 python tools/solver_bench.py --n 256 --b 1024 --iters 10 --mode f32 --reps 2 2>&1 | grep "\[gemm\].*10240" | sort | uniq -c | sort -rn | head -1; env "$@" timeout 300 python tools/solver_bench.py --n 256 --b 1024 --iters 10 --mode f32 | grep "ndb"; }
for l in 0 1 0 1; do echo "== lean $l"; run DASH_LEAN=$l; done
