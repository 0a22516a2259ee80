# Evidence for one round (on the GPU box): GPU tests, the bench line, the reference arm, the launch
# list of one T step and of one C4 step, and ncu --set full captures of the FP64 downdate at T and the
# rqb_svd Jacobi kernels.   usage: bash tools/evidence.sh r02
R=${1:-r02}
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gputests_$R.log 2>&1; echo tests_rc=$?
timeout 900 python bench.py > gpurun_out/bench_$R.json 2> gpurun_out/bench_$R.err; echo bench_rc=$?
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_$R.json 2> gpurun_out/bench_ref_$R.err; echo ref_rc=$?
timeout 600 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-post --records none \
    > gpurun_out/plain_$R.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$R.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-post --records none \
    > gpurun_out/ncu_launch_$R.log 2>&1; echo launches_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4_$R.csv \
    env PYTHONPATH=. python tools/factor_once.py C4 2 > gpurun_out/ncu_launch_c4_$R.log 2>&1; echo c4_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k "regex:gemm_f64_kernelILi0ELi64ELi2E" -s 3 -c 1 -o gpurun_out/prof_down_$R \
    env PYTHONPATH=. python tools/quick_run.py T 1 > gpurun_out/ncu_down_$R.log 2>&1; echo down_rc=$?
# qb_pivoted_qr at T: launch list (after an uninstrumented run) and one persistent panel launch under --set full
PYTHONPATH=. timeout 300 python tools/qrcp_once.py T > gpurun_out/qrcp_plain_$R.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_qrcp_$R.csv \
    env PYTHONPATH=. python tools/qrcp_once.py T > gpurun_out/ncu_launch_qrcp_$R.log 2>&1; echo qrcp_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k "regex:qrcp_panel_kernel" -s 90 -c 1 -o gpurun_out/prof_qrcp_$R \
    env PYTHONPATH=. python tools/qrcp_once.py T > gpurun_out/ncu_qrcp_$R.log 2>&1; echo qrcp_full_rc=$?
