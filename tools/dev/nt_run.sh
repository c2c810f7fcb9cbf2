cd $GRAFT_REPO_ROOT
run() { env "$@" DASH_GEMM_DEBUG=2 timeout 300 python tools/solver_bench.py --n 256 --b 1024 --iters 10 --mode f32 --reps 2 2>&1 | grep "\[gemm\].*10240" | sort | uniq -c | sort -rn | head -1; env "$@" timeout 300 python tools/solver_bench.py --n 256 --b 1024 --iters 10 --mode f32 | grep "ndb: total"; }
for e in 0 192 32 224 8 200; do echo "== exp $e"; run DASH_EXP=$e; done
