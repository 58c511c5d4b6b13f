mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest13.log 2>&1; echo pytest=$?
for c in cfg2_2d_N1024_sweep cfg5_2d_N2048_darcy; do
for k in 0 1; do
DD_NO_COMPACT=$k timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench13_${c}_nocompact$k.json 2>&1; echo b=$?
done; done
