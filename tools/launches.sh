# ncu launch list of the bench command; usage: bash tools/launches.sh <tag>
R=${1:-r01}
python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-post > gpurun_out/plain_$R.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$R.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-post > gpurun_out/ncu_launch_$R.log 2>&1
echo launches_rc=$?
grep -o '"gpu_launches": [0-9]*' gpurun_out/plain_$R.log
