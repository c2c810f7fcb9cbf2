# A/B on one box: current library vs build/libdash_b200_prev.so (k-block-granular ring issue loop)
for i in 1 2; do
for lib in paper_2602_02016_b200/libdash_b200.so build/libdash_b200_prev.so; do echo "== $lib"; DASH_LIB=$lib timeout 300 python tools/solver_bench.py --n 1820 --b 1024 --mode f32 --reps 2 2>&1 | grep "ndb: total"; done
done
for lib in paper_2602_02016_b200/libdash_b200.so build/libdash_b200_prev.so paper_2602_02016_b200/libdash_b200.so; do echo "== bench $lib"; DASH_LIB=$lib python bench.py --steps 4 --warmup 3 --no-cpu --no-e2e --no-parity 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['phases_ms'], d['clocks']['sm_mhz'])"; done
