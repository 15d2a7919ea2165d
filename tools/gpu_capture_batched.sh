set -x
CMD="python bench.py --no-cpu --window-only --steps 6 --warmup 8"
export IPC_LOOP_GRAPH=0
$CMD > gpurun_out/plain_cap.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "bench_timed/" -k regex:"k_ls_value" -c 3 -o /tmp/cap $CMD > gpurun_out/ncu_cap.log 2>&1
ncu -i /tmp/cap.ncu-rep --page raw --csv > gpurun_out/cap_raw.csv
for k in k_ls_value; do
  ncu -i /tmp/cap.ncu-rep --page source --csv --print-source cuda,sass -k regex:$k -c 1 > gpurun_out/cap_src_$k.csv 2>&1
done
ls -la gpurun_out
