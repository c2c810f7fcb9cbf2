cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
run() { env "$@" DASH_GEMM_DEBUG=2 timeout 300 python tools/solver_bench.py --n 256 --b 1024 --iters 10 --mode f32 --reps 2 2>&1 | grep "\[gemm\].*10240" | sort | uniq -c | sort -rn | head -1; env "$@" timeout 300 python tools/solver_bench.py --n 256 --b 1024 --iters 10 --mode f32 | grep "ndb"; }
for u in 0 1 0 1; do echo "== up $u"; run DASH_NDB_UP=$u; done
echo "== up f16"; timeout 300 python tools/solver_bench.py --n 256 --b 1024 --iters 10 --mode f16 | grep "ndb: total"
echo "== noup f16"; DASH_NDB_UP=0 timeout 300 python tools/solver_bench.py --n 256 --b 1024 --iters 10 --mode f16 | grep "ndb: total"
