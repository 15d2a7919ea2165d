# A/B of library builds on the config-3 bench (W5 K20): plain runs (R repeats, interleaved) + one per-kernel profile each
R=${R:-2}
for i in $(seq $R); do for L in "$@"; do
  IPC_B200_LIB=$PWD/$L python bench.py --no-cpu --no-closed-loop --steps 20 --warmup 5 > gpurun_out/ab_${L}_$i.json 2> gpurun_out/ab_${L}_$i.err
done; done
for L in "$@"; do
  IPC_B200_LIB=$PWD/$L BENCH_PROFILE=2 python bench.py --no-cpu --no-closed-loop --steps 20 --warmup 5 > gpurun_out/abp_$L.json 2> gpurun_out/abp_$L.err
done
