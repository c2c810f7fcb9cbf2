python tools/solver_bench.py --solver cheb --n 1820 --b 1024 --mode f16 --reps 2 2>&1 | grep "cheb"
python tools/solver_bench.py --solver cheb --n 1820 --b 1024 --mode f32 --reps 2 2>&1 | grep "cheb: total"
python tools/solver_bench.py --n 1820 --b 1024 --mode f16 --reps 2 2>&1 | grep "ndb: total"
python tools/solver_bench.py --n 1820 --b 1024 --mode f32 --reps 2 2>&1 | grep "ndb: total"
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
