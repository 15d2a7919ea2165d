for i in 1 2; do for T in 370 444 518; do
  IPC_TAIL=$T python bench.py --no-cpu --no-closed-loop --steps 20 --warmup 5 > gpurun_out/ab_u${T}_$i.json 2>&1
done; done
