# ncu evidence for one round: launch list of the bench command + full sections of the 3 big GEMMs.
# usage (on the GPU box): bash tools/prof.sh r01
R=${1:-r01}
python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-post > gpurun_out/plain_$R.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$R.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-post > gpurun_out/ncu_launch_$R.log 2>&1
echo launches_rc=$?
PYTHONPATH=. python tools/quick_run.py T 1 > gpurun_out/plain2_$R.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k "regex:gemm_f64_kernelILi0ELi64ELi2E" -c 1 -o gpurun_out/prof_down_$R \
    env PYTHONPATH=. python tools/quick_run.py T 1 > gpurun_out/ncu_full_$R.log 2>&1
echo full_rc=$?
ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k "regex:gemm_f64_kernelILi(0ELi64ELi0|1ELi64ELi1)E" -c 2 -o gpurun_out/prof_yb_$R \
    env PYTHONPATH=. python tools/quick_run.py T 1 > gpurun_out/ncu_full2_$R.log 2>&1
echo full2_rc=$?
