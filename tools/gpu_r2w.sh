mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/w2_build.log 2>&1; echo build=$?
for c in cfg2_2d_N1024_sweep cfg5_2d_N2048_darcy; do
DD_PHASE_TIMING=1 timeout 300 python tools/prof_step.py --config $c --solves 3 2>&1 | grep "\[dd" | tail -3
DD_PHASE_TIMING=1 DD_NO_GRAPH=1 timeout 300 python tools/prof_step.py --config $c --solves 3 2>&1 | grep "\[dd" | tail -3
done
