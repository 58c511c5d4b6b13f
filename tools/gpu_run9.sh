mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest9.log 2>&1; echo pytest=$?
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench9_cfg2.json 2>gpurun_out/bench9_cfg2.err; echo b=$?
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --frac-mode ra > gpurun_out/bench9_cfg2_ra.json 2>&1; echo b=$?
timeout 600 python bench.py --steps 3 --warmup 1 --mode bulk > gpurun_out/bench9_cfg2_bulk.json 2>&1; echo b=$?
