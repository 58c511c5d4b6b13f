# packed-symmetric F stream (cfg4): launch list of its two kernels + a full capture of k_fx_sym
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/y_build.log 2>&1; echo build=$?
export DD_NO_GRAPH=1 DD_FX_PACKED=1
timeout 300 python tools/prof_step.py --config cfg4_3d_N128 --solves 1 > gpurun_out/y_pstep.log 2>&1; echo pstep=$?
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,lts__t_bytes.sum --clock-control none --csv -k regex:"k_fx_sym|k_cheb" \
  --log-file gpurun_out/y_launches_cfg4.csv python tools/prof_step.py --config cfg4_3d_N128 --solves 1 > gpurun_out/y_ncu_launch.log 2>&1; echo ncu_launch=$?
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_fx_sym" -s 6 -c 2 \
    -o gpurun_out/y_full_fxsym -f python tools/prof_step.py --config cfg4_3d_N128 --solves 1 > gpurun_out/y_ncu_full.log 2>&1; echo ncu_full=$?
