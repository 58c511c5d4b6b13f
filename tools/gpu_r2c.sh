# pole-sum v2 phases + ncu (tool)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c_build.log 2>&1; echo build=$?
for c in cfg2_2d_N1024_sweep cfg5_2d_N2048_darcy; do
  DD_PHASE_TIMING=1 DD_NO_GRAPH=1 timeout 300 python tools/prof_step.py --config $c --solves 2 > gpurun_out/c_phase_$c.log 2>&1
  DD_POLESUM_V1=1 DD_PHASE_TIMING=1 DD_NO_GRAPH=1 timeout 300 python tools/prof_step.py --config $c --solves 2 > gpurun_out/c_phase_v1_$c.log 2>&1
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_pcg_iter -s 20 -c 1 -o gpurun_out/c_pcg_iter_cfg5 python tools/prof_step.py --config cfg5_2d_N2048_darcy --solves 2 > gpurun_out/c_ncu.log 2>&1; echo ncu=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_pcg_iter -s 20 -c 1 -o gpurun_out/c_pcg_iter_cfg2 python tools/prof_step.py --config cfg2_2d_N1024_sweep --solves 2 > gpurun_out/c_ncu2.log 2>&1; echo ncu2=$?
