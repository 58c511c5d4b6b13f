mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/z_build.log 2>&1; echo build=$?
timeout 900 python -m pytest tests/test_gpu_3d.py -x -q -p no:cacheprovider -k "packed" > gpurun_out/z_pytest.log 2>&1; echo pytest=$?
tail -1 gpurun_out/z_pytest.log
export DD_NO_GRAPH=1
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv -k regex:"k_fx_sym" \
  --log-file gpurun_out/z_launches.csv python tools/prof_step.py --config cfg4_3d_N128 --solves 1 > gpurun_out/z_ncu.log 2>&1; echo ncu=$?
