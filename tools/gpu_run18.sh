mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python bench.py --config cfg4_3d_N128 --frac-mode ra --steps 3 --warmup 3 > gpurun_out/bench18_cfg4_ra.json 2> gpurun_out/bench18_cfg4_ra.err; echo b=$?
timeout 900 python bench.py --mode bulk-pcg --config cfg1_2d_N32 --steps 5 --warmup 3 > gpurun_out/bench18_bulkpcg_cfg1.json 2>&1; echo b2=$?
timeout 900 python bench.py --mode bulk-pcg --steps 2 --warmup 1 > gpurun_out/bench18_bulkpcg_cfg2.json 2>&1; echo b3=$?
timeout 600 python bench.py --t 0.25 --shifted --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench18_t025.json 2>&1; echo b4=$?
