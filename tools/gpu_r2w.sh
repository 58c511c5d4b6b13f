mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/w2_build.log 2>&1; echo build=$?
for sk in 0 1 2 4 3 5 6 7; do DD_V2_SKIP=$sk python tools/time_precond.py --config cfg5_2d_N2048_darcy 2>&1 | tail -1; done
for sk in 0 7; do DD_V2_SKIP=$sk python tools/time_precond.py --config cfg2_2d_N1024_sweep 2>&1 | tail -1; done
