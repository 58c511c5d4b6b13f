mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
#timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest8.log 2>&1; echo pytest=$?
for m in 0 1; do
DD_NO_MERGED=$m DD_PHASE_TIMING=1 timeout 120 python tools/prof_step.py --solves 3 2>&1 | grep cycles | tail -2 > gpurun_out/phase8_m$m.log
for c in cfg2_2d_N1024_sweep cfg3_2d_N4096 cfg5_2d_N2048_darcy; do
DD_NO_MERGED=$m timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench8_m${m}_$c.json 2>/dev/null; echo b=$?
done; done
