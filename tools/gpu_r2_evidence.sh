# Round-2 evidence pass (tool; under gpurun from the repo root): GPU suite, smoke, bench lines for
# every config and mode, the ncu launch list of the default bench command, ncu --set full captures.
mkdir -p gpurun_out/ev
O=gpurun_out/ev
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?
timeout 1200 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo bench_default=$?
for c in cfg2_2d_N1024_sweep cfg3_2d_N4096 cfg1_2d_N32 cfg5i_2d_N2048_darcy_rtol1e-5; do
  timeout 900 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err; echo bench $c=$?
done
timeout 1500 python bench.py --config cfg4_3d_N128 > $O/bench_cfg4.json 2> $O/bench_cfg4.err; echo bench cfg4=$?
timeout 900 python bench.py --config cfg4_3d_N128 --frac-mode ra --no-cpu-baseline > $O/bench_cfg4_ra.json 2> $O/bench_cfg4_ra.err; echo bench cfg4ra=$?
timeout 900 python bench.py --config cfg2_2d_N1024_sweep --frac-mode ra --no-cpu-baseline > $O/bench_cfg2_ra.json 2> $O/bench_cfg2_ra.err; echo bench cfg2ra=$?
timeout 1500 python bench.py --no-cpu-baseline --emulate-ranks 8 > $O/bench_cfg5_em8.json 2> $O/bench_cfg5_em8.err; echo em5=$?
timeout 1500 python bench.py --config cfg4_3d_N128 --no-cpu-baseline --emulate-ranks 8 > $O/bench_cfg4_em8.json 2> $O/bench_cfg4_em8.err; echo em4=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err; echo ref=$?
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv \
  --log-file $O/launches_cfg5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1; echo ncu_launch=$?
export DD_NO_GRAPH=1
for c in cfg5_2d_N2048_darcy cfg2_2d_N1024_sweep; do
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_dgemm|k_pcg_iter" -s 8 -c 2 \
      -o $O/full_$c -f python tools/prof_step.py --config $c --solves 2 > $O/ncu_$c.log 2>&1; echo ncu $c=$?
done
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_cheb_step|k_fx_sym" -s 6 -c 3 \
    -o $O/full_cfg4 -f python tools/prof_step.py --config cfg4_3d_N128 --solves 1 > $O/ncu_cfg4.log 2>&1; echo ncu cfg4=$?
# per-iteration launch list of one config-5 solve outside the graph (GEMM / fused PCG vs live columns)
DD_NO_GRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches_cfg5_nograph.csv python tools/prof_step.py --config cfg5_2d_N2048_darcy --solves 2 > $O/ncu_nograph.log 2>&1; echo ncu_nograph=$?
