# usage: bash tools/prof_one.sh <tag> <mangled-regex> <count> [skip]
T=$1; RX=$2; C=${3:-1}; S=${4:-0}
PYTHONPATH=. python tools/quick_run.py T 1 > gpurun_out/plain_$T.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k "regex:$RX" -s $S -c $C \
    -o gpurun_out/prof_$T env PYTHONPATH=. python tools/quick_run.py T 1 > gpurun_out/ncu_$T.log 2>&1
echo rc=$?
