for i in 1 2; do
  IPC_B200_LIB=$PWD/exp_pdl_lib.so python bench.py --no-cpu --no-closed-loop --steps 20 --warmup 5 > gpurun_out/ab_pdlon_$i.json 2>&1
  IPC_PDL=0 IPC_B200_LIB=$PWD/exp_pdl_lib.so python bench.py --no-cpu --no-closed-loop --steps 20 --warmup 5 > gpurun_out/ab_pdloff_$i.json 2>&1
done
