# cfg4 inner-loop kernels: launch list of the matched kernels + full captures (Chebyshev, parity-blocked D̂)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/y_build.log 2>&1; echo build=$?
export DD_NO_GRAPH=1
timeout 300 python tools/prof_step.py --config cfg4_3d_N128 --solves 2 > gpurun_out/y_pstep.log 2>&1; echo pstep=$?
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:"k_dgemm_tile|k_inner|k_dgemm_streamk" \
  --log-file gpurun_out/y_launches_cfg4.csv python tools/prof_step.py --config cfg4_3d_N128 --solves 2 > gpurun_out/y_ncu_launch.log 2>&1; echo ncu_launch=$?
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_dgemm_tile" -s 400 -c 4 \
    -o gpurun_out/y_full_cfg4 -f python tools/prof_step.py --config cfg4_3d_N128 --solves 2 > gpurun_out/y_ncu_full.log 2>&1; echo ncu_full=$?
