# Evidence pass (tool; under gpurun from the repo root): ncu --set full of the final dominant
# kernels — grouped GEMM + fused PCG kernel (cfg2, cfg5), the 3D F stream and inner-CG update (cfg4).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/g_build.log 2>&1
export DD_NO_GRAPH=1
for c in cfg2_2d_N1024_sweep cfg5_2d_N2048_darcy; do
  timeout 300 python tools/prof_step.py --config $c --solves 2 > gpurun_out/g_plain_$c.log 2>&1 && \
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_dgemm|k_pcg_iter" -s 8 -c 3 \
      -o gpurun_out/g_full_$c -f python tools/prof_step.py --config $c --solves 2 > gpurun_out/g_ncu_$c.log 2>&1; echo ncu $c=$?
done
timeout 300 python tools/prof_step.py --config cfg4_3d_N128 --solves 1 > gpurun_out/g_plain_cfg4.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_dgemm_streamk|k_inner_update" -s 4 -c 3 \
    -o gpurun_out/g_full_cfg4 -f python tools/prof_step.py --config cfg4_3d_N128 --solves 1 > gpurun_out/g_ncu_cfg4.log 2>&1; echo ncu cfg4=$?
