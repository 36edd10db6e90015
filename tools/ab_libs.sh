# Same-box A/B of library builds: bash tools/ab_libs.sh <lib-suffix> ... (paper_0805_3041_b200/libgmg_<suffix>.so);
# alternates the builds twice (box-to-box variation is ~3%, so only same-call comparisons count).
cd $GRAFT_REPO_ROOT
P='import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(sys.argv[1], sys.argv[2], "ms", round(d["ms_per_step"],4))'
for rep in 1 2; do for s in "$@"; do
  for wl in C4 C5; do
    GMG_LIB_PATH=$PWD/paper_0805_3041_b200/libgmg_$s.so python bench.py --workload $wl --steps $([ $wl = C4 ] && echo 20 || echo 10) --warmup 5 --e2e-steps 0 --no-cpu-baseline --no-c5 --no-per-level 2>/dev/null | python -c "$P" $s $wl
  done
done; done
