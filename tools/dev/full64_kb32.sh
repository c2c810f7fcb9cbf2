# FULL64 on the K-block 32 kernel with one ring unit per K block: accuracy (C1 fixed-10, floor probe) and speed
PREC=f64 timeout 300 python tools/dev/diag_c1_fixed.py 2>&1 | grep -E "group|update"
timeout 600 python tools/floor_probe.py --kmax 12 --mode f64 2>&1 | grep -A2 "B=1024 cond=100$\|B=1024 cond=10$"
timeout 300 python tools/solver_bench.py --n 1820 --b 1024 --mode f64 --reps 1 2>&1 | grep "ndb: total"
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_boundary.py tests/test_gpu_parity.py -q -s -k "c1 or default" 2>&1 | grep -E "relF|passed|failed"
timeout 300 python tools/solver_bench.py --n 1820 --b 1024 --mode f32 --reps 1 2>&1 | grep "ndb: total"
timeout 300 python tools/floor_probe.py --kmax 11 --mode f64 2>&1 | grep -A2 "B=256 cond=100$\|C1 literal"
