# Final state: GPU suite, smoke, bench lines (2D configs), launch list of the default bench, cfg5 fused-PCG capture.
mkdir -p gpurun_out/f2; O=gpurun_out/f2
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?
timeout 1200 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo bench_default=$?
for c in cfg2_2d_N1024_sweep cfg3_2d_N4096 cfg1_2d_N32 cfg5i_2d_N2048_darcy_rtol1e-5; do
  timeout 900 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err; echo bench $c=$?
done
timeout 900 python bench.py --config cfg2_2d_N1024_sweep --frac-mode ra --no-cpu-baseline > $O/bench_cfg2_ra.json 2> $O/bench_cfg2_ra.err; echo cfg2ra=$?
timeout 1500 python bench.py --no-cpu-baseline --emulate-ranks 8 > $O/bench_cfg5_em8.json 2> $O/bench_cfg5_em8.err; echo em5=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err; echo ref=$?
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv \
  --log-file $O/launches_cfg5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1; echo ncu_launch=$?
DD_NO_GRAPH=1 timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_dgemm|k_pcg_iter" -s 8 -c 2 \
    -o $O/full_cfg5 -f python tools/prof_step.py --config cfg5_2d_N2048_darcy --solves 2 > $O/ncu_cfg5.log 2>&1; echo ncu cfg5=$?
