for L in exp_head_lib.so exp_new_lib.so; do
  IPC_B200_LIB=$PWD/$L IPC_TAIL=0 python bench.py --no-cpu --no-closed-loop --steps 20 --warmup 5 > gpurun_out/ab_notail_${L}_1.json 2>&1
done
R=2 bash tools/ab_libs.sh exp_head_lib.so exp_new_lib.so
