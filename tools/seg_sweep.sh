# sweep of the rows-per-segment choice for the two largest C4 levels (GMG_SEG_FORCE), same box
cd $GRAFT_REPO_ROOT
P='import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(sys.argv[1], "ms", round(d["ms_per_step"],4), "roof", round(d["roofline"]["frac"],3))'
for f in "" "8191:64" "8191:120" "8191:128" "8191:86" "4095:32" "4095:64" "4095:22" "8191:64,4095:64" "8191:120,4095:64,2047:32"; do
  GMG_SEG_FORCE="$f" python bench.py --workload C4 --steps 20 --warmup 5 --e2e-steps 0 --no-cpu-baseline --no-c5 --no-per-level 2>/dev/null | python -c "$P" "force[$f]"
done
