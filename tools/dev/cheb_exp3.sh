for x in 0 512; do echo "== DASH_EXP=$x"; DASH_EXP=$x python tools/solver_bench.py --solver cheb --n 1820 --b 1024 --mode f16 --reps 2 2>&1 | grep "cheb: total"; DASH_EXP=$x python tools/solver_bench.py --solver cheb --n 1820 --b 1024 --mode f32 --reps 2 2>&1 | grep "cheb: total"; done
python tools/step_profile.py 2>&1 | grep -E "tiles=  38304|accumulated"
DASH_EXP=512 python tools/step_profile.py 2>&1 | grep -E "tiles=  38304|accumulated"
