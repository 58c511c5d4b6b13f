mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest7.log 2>&1; echo pytest=$?
DD_PHASE_TIMING=1 timeout 120 python tools/prof_step.py --solves 3 > gpurun_out/phase7_cfg2.log 2>&1
for c in cfg2_2d_N1024_sweep cfg3_2d_N4096 cfg5_2d_N2048_darcy; do
timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench7_$c.json 2>gpurun_out/bench7_$c.err; echo b=$?
done
