# one full capture of the fused Chebyshev step (cfg4)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/y_build.log 2>&1; echo build=$?
export DD_NO_GRAPH=1
timeout 300 python tools/prof_step.py --config cfg4_3d_N128 --solves 2 > gpurun_out/y_pstep.log 2>&1; echo pstep=$?
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_cheb_step" -s 100 -c 1 \
    -o gpurun_out/y_full_cheb -f python tools/prof_step.py --config cfg4_3d_N128 --solves 2 > gpurun_out/y_ncu_full.log 2>&1; echo ncu_full=$?
