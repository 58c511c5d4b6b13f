# shared-pair grouped GEMM: parity + ncu (tool)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/h_build.log 2>&1; echo build=$?
timeout 900 python -m pytest tests/test_gpu_r2.py tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "pair or full_config" > gpurun_out/h_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/h_pytest.log
DD_NO_GRAPH=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_dgemm_pair -s 5 -c 1 -o gpurun_out/h_pair_cfg5 python tools/prof_step.py --config cfg5_2d_N2048_darcy --solves 2 > gpurun_out/h_ncu.log 2>&1; echo ncu=$?
