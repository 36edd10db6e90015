# Source-level (SASS) stall samples of one kernel launch: bash tools/ncu_source.sh <name> <kernel-regex> <launch-skip> <command...>
# -> gpurun_out/<name>.sass.csv (read with tools/ncu_top_stalls.py)
name=$1; kre=$2; skip=$3; shift 3
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k "regex:$kre" --launch-skip "$skip" -c 1 -o /tmp/$name -f "$@" > gpurun_out/$name.ncu.log 2>&1
ncu -i /tmp/$name.ncu-rep --page source --csv --print-source sass > gpurun_out/$name.sass.csv 2>&1
