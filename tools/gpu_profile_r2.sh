# Round-2 evidence pass (tool; under gpurun from the repo root): the ncu launch list of the default
# bench command (config 5) and ncu --set full captures of the dominant kernels (cfg5, cfg2, cfg4).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/p2_build.log 2>&1; echo build=$?
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/p2_gpu.txt
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/p2_plain.log 2>&1; echo plain=$?
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv \
  --log-file gpurun_out/p2_launches_cfg5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/p2_ncu_launch.log 2>&1; echo ncu_launch=$?
export DD_NO_GRAPH=1
for c in cfg5_2d_N2048_darcy cfg2_2d_N1024_sweep; do
  timeout 300 python tools/prof_step.py --config $c --solves 2 > gpurun_out/p2_pstep_$c.log 2>&1 && \
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_dgemm|k_pcg_iter" -s 8 -c 2 \
      -o gpurun_out/p2_full_$c -f python tools/prof_step.py --config $c --solves 2 > gpurun_out/p2_ncu_$c.log 2>&1; echo ncu $c=$?
done
timeout 300 python tools/prof_step.py --config cfg4_3d_N128 --solves 1 > gpurun_out/p2_pstep_cfg4.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_dgemm_streamk|k_inner_update" -s 4 -c 3 \
    -o gpurun_out/p2_full_cfg4 -f python tools/prof_step.py --config cfg4_3d_N128 --solves 1 > gpurun_out/p2_ncu_cfg4.log 2>&1; echo ncu cfg4=$?
