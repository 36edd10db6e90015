# sweep of the rows-per-segment choice per level width (GMG_SEG_FORCE), same box; C4 ms per cycle
cd $GRAFT_REPO_ROOT
P='import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(sys.argv[1], "ms", round(d["ms_per_step"],4))'
for f in "" "2047:16" "2047:32" "2047:64" "1023:16" "1023:32" "511:16" "511:32" "255:16" "4095:64,2047:32,1023:16" "4095:64,2047:16,1023:16,511:16" ""; do
  GMG_SEG_FORCE="$f" python bench.py --workload C4 --steps 20 --warmup 5 --e2e-steps 0 --no-cpu-baseline --no-c5 --no-per-level 2>/dev/null | python -c "$P" "force[$f]"
done
