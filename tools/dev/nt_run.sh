cd $GRAFT_REPO_ROOT
for cfg in "DASH_EXP=0" "DASH_EXP=2" "DASH_EXP=4" "DASH_EXP=8" "DASH_NT=128 DASH_EXP=2"; do
  echo "== $cfg f16"; env $cfg timeout 300 python tools/solver_bench.py --n 256 --b 1024 --iters 10 --mode f16 | grep "ndb: total"
done
echo "== f32 exp2"; DASH_EXP=2 timeout 300 python tools/solver_bench.py --n 256 --b 1024 --iters 10 --mode f32 | grep "ndb: total"
echo "== f32 exp2 wide"; DASH_NT=2562 DASH_EXP=2 timeout 300 python tools/solver_bench.py --n 256 --b 1024 --iters 10 --mode f32 | grep "ndb: total"
timeout 600 python bench.py --precision f16 --no-cpu --steps 5 --warmup 3
timeout 600 python bench.py --precision f16 --solver cbshv --no-cpu --steps 5 --warmup 3
DASH_NT=128 timeout 600 python bench.py --precision f16 --solver cbshv --no-cpu --no-e2e --steps 5 --warmup 3
