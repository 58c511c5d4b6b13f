mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_frac.py -x -q > gpurun_out/pytest16.log 2>&1; echo pytest=$?
DD_PHASE_TIMING=1 timeout 120 python tools/prof_step.py --solves 3 2>&1 | grep cycles | tail -2 > gpurun_out/phase16.log
for c in cfg2_2d_N1024_sweep cfg5_2d_N2048_darcy cfg3_2d_N4096; do
for k in 0 1; do
DD_NO_PAIR=$k timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench16_${c}_nopair$k.json 2>&1; echo b=$?
done; done
