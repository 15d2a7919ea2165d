# Round evidence on the GPU box: headline bench (driver's W5/K20 window),
# W3 window, reference arm, the ncu window capture of the dominant kernel
# (fp64 instruction counts over exactly the timed launches) and the launch
# list of the window (host-loop mode so that graph-body kernels are listed).
set -x
python bench.py --steps 20 --warmup 5 > gpurun_out/ev_bench_w5.json 2> gpurun_out/ev_bench_w5.err
python bench.py --no-cpu --no-closed-loop --steps 20 --warmup 3 > gpurun_out/ev_bench_w3.json 2> gpurun_out/ev_bench_w3.err
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ev_ref_w5.json 2> gpurun_out/ev_ref_w5.err
CMD="python bench.py --no-cpu --window-only --steps 20 --warmup 5"
$CMD > gpurun_out/ev_window_plain.log 2>&1 && \
ncu -f --set full --metrics sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum \
    --clock-control none --nvtx --nvtx-include "bench_timed/" -k regex:k_env_newton_rest -o /tmp/ev_window $CMD > gpurun_out/ev_ncu_window.log 2>&1
ncu -i /tmp/ev_window.ncu-rep --page raw --csv > gpurun_out/ev_window_raw.csv
IPC_LOOP_GRAPH=0 $CMD > gpurun_out/ev_ll_plain.log 2>&1 && \
IPC_LOOP_GRAPH=0 ncu -f --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "bench_timed/" --csv --log-file gpurun_out/ev_launches.csv $CMD > gpurun_out/ev_ncu_ll.log 2>&1
ls -la gpurun_out | grep ev_
