# Same-box A/B of library builds: bash tools/ab_libs.sh <lib-suffix> ... (paper_0805_3041_b200/libgmg_<suffix>.so;
# build variants with GMG_EXTRA_NVFLAGS/GMG_BUILD_DIR/GMG_LIB_OUT). AB_ENV="VAR=val" adds a run of the first
# library under that environment. Builds are deterministic (no -split-compile): one pass is enough.
cd $GRAFT_REPO_ROOT
P='import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(sys.argv[1], sys.argv[2], "ms", round(d["ms_per_step"],4))'
run() { for wl in C4 C5; do
    env $2 GMG_LIB_PATH=$PWD/paper_0805_3041_b200/libgmg_$1.so python bench.py --workload $wl --steps $([ $wl = C4 ] && echo 20 || echo 10) --warmup 5 --e2e-steps 0 --no-cpu-baseline --no-c5 --no-per-level 2>/dev/null | python -c "$P" "$1[$2]" $wl
  done; }
for s in "$@"; do run $s "X=1"; done
for e in $AB_ENV; do run $1 "$e"; done
run $1 "X=1"
