cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "power_iteration" 2>&1 | tail -2
for b in 1024 512 256; do echo "== new b=$b"; timeout 300 python tools/pi_bench.py --n 296 --b $b --iters 30 --tc 2>&1 | tail -2; done
cp paper_2602_02016_b200/libdash_b200.so /tmp/new.so; cp build/old/libdash_b200.so paper_2602_02016_b200/libdash_b200.so
for b in 1024 512 256; do echo "== old b=$b"; timeout 300 python tools/pi_bench.py --n 296 --b $b --iters 30 --tc 2>&1 | tail -2; done
cp /tmp/new.so paper_2602_02016_b200/libdash_b200.so
timeout 600 python bench.py --no-cpu > gpurun_out/bench_pi.json 2>/dev/null; tail -1 gpurun_out/bench_pi.json | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['clocks'], d['phases_ms'], d['e2e']['value'])"
