mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
DD_PHASE_TIMING=1 timeout 120 python tools/prof_step.py --solves 3 > gpurun_out/phase6_cfg2.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest6.log 2>&1; echo pytest=$?
for pdl in 0 1; do
DD_NO_PDL=$pdl timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench6_nopdl$pdl.json 2>&1; echo b=$?
done
timeout 300 python bench.py --config cfg3_2d_N4096 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench6_cfg3.json 2>&1
