# ncu --set full capture of one kernel launch, exported to text (the .ncu-rep stays on the box
# unless KEEP_REP=1). Usage: bash tools/ncu_capture.sh <name> <kernel-regex> <launch-skip> <command...>
name=$1; kre=$2; skip=$3; shift 3
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k "regex:$kre" --launch-skip "$skip" -c 1 \
    -o /tmp/$name -f "$@" > gpurun_out/$name.ncu.log 2>&1
ncu -i /tmp/$name.ncu-rep --page details --csv > gpurun_out/$name.details.csv 2>&1
ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/$name.raw.csv 2>&1
ncu -i /tmp/$name.ncu-rep --page source --csv --print-source sass > gpurun_out/$name.sass.csv 2>&1
[ "$KEEP_REP" = 1 ] && cp /tmp/$name.ncu-rep gpurun_out/
true
