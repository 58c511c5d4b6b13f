# Evidence pass for the grouped Schur apply (tool; run under gpurun from the repo root):
# ncu --set full of the grouped GEMM (cfg2: cluster split-K tile kernel; cfg5/cfg3: stream-K) and
# the fused pole-sum kernel, then the launch list of the headline bench command.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/f_build.log 2>&1
export DD_NO_GRAPH=1
for c in cfg2_2d_N1024_sweep cfg5_2d_N2048_darcy cfg3_2d_N4096; do
  timeout 300 python tools/prof_step.py --config $c --solves 2 > gpurun_out/f_plain_$c.log 2>&1 && \
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_dgemm|k_pcg_iter" -s 8 -c 3 \
      -o gpurun_out/f_full_$c -f python tools/prof_step.py --config $c --solves 2 > gpurun_out/f_ncu_$c.log 2>&1; echo ncu $c=$?
done
unset DD_NO_GRAPH
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/f_plain.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/f_launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/f_ncu_launch.log 2>&1; echo ncu_launch=$?
