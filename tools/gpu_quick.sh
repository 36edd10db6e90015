# quick GPU check: parity suite + one bench line (no e2e / cpu legs)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
for i in 1 2; do
python bench.py --steps 20 --warmup 5 --e2e-steps 0 --no-cpu-baseline --no-c5 --no-per-level 2>/dev/null | python -c 'import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print("C4 ms", d["ms_per_step"], "roofline", d["roofline"]["frac"])'
done
python bench.py --workload C5 --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-c5 --no-per-level 2>/dev/null | python -c 'import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print("C5 ms", d["ms_per_step"])'
