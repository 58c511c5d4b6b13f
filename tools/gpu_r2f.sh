# pole-sum v2.1 check (tool)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/f_build.log 2>&1; echo build=$?
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_r2.py -x -q -p no:cacheprovider -k "not 3d and not cfg4" > gpurun_out/f_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/f_pytest.log
for c in cfg2_2d_N1024_sweep cfg5_2d_N2048_darcy cfg3_2d_N4096; do
  DD_PHASE_TIMING=1 DD_NO_GRAPH=1 timeout 300 python tools/prof_step.py --config $c --solves 2 > gpurun_out/f_phase_$c.log 2>&1
done
DD_NO_GRAPH=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_pcg_iter -s 20 -c 1 -o gpurun_out/f_pcg_iter_cfg2 python tools/prof_step.py --config cfg2_2d_N1024_sweep --solves 2 > gpurun_out/f_ncu2.log 2>&1; echo ncu2=$?
