# A/B of older builds (git worktrees under ab/, each with its own libgmg_b200.so) against HEAD
cd $GRAFT_REPO_ROOT
P='import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(sys.argv[1], "ms", d["ms_per_step"])'
for t in ${AB_TREES:-r1}; do
 (cd ab/$t && python bench.py --steps 20 --warmup 5 --e2e-steps 0 --no-cpu-baseline $(python bench.py --help | grep -q no-c5 && echo --no-c5 --no-per-level) 2>/dev/null | python -c "$P" $t)
done
python bench.py --steps 20 --warmup 5 --e2e-steps 0 --no-cpu-baseline --no-c5 --no-per-level 2>/dev/null | python -c "$P" HEAD
