# Config 2 (10,368-tet soft cube in the gripper): per-step kernel times and
# PCG iterations, then the launch list and a full capture of the PCG kernel
# and the library sort/scan launches of the sparse assembly (run on the GPU box)
set -x
timeout 900 python tools/config2_steps.py 12 30 > gpurun_out/c2_steps.jsonl 2> gpurun_out/c2_steps.err || exit 1
CMD="python tools/config2_steps.py 12 5"
$CMD > gpurun_out/c2_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none -s 2000 -c 3000 --csv --log-file gpurun_out/c2_launches.csv $CMD > gpurun_out/c2_ncu_l.log 2>&1
ncu --set full --clock-control none -k regex:"k_pcg_coop|DeviceRadixSort|DeviceScan|k_asm" -s 200 -c 12 -o /tmp/c2 $CMD > gpurun_out/c2_ncu_f.log 2>&1
ncu -i /tmp/c2.ncu-rep --page raw --csv > gpurun_out/c2_raw.csv
ls -la gpurun_out | head -40
