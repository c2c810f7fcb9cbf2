cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for u in 0 1; do echo "== up $u cn"; DASH_NDB_UP=$u timeout 600 python bench.py --solver cn --no-cpu --no-e2e --steps 3 --warmup 3 2>/dev/null | python3 -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['clocks']['sm_mhz'], d['roofline']['achieved'], d['phases_ms'])"; done
