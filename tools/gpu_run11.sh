mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_frac_ra.py -x -q > gpurun_out/pytest11.log 2>&1; echo pytest=$?
for c in cfg2_2d_N1024_sweep cfg5_2d_N2048_darcy cfg3_2d_N4096 cfg5i_2d_N2048_darcy_rtol1e-5; do
for k in 0 1; do
DD_NO_SKIP=$k timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench11_${c}_noskip$k.json 2>&1; echo b=$?
done; done
