mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/l_build.log 2>&1; echo build=$?
for c in cfg5_2d_N2048_darcy cfg2_2d_N1024_sweep; do for m in 0 1 2 4 7; do
  DD_V2_SKIP=$m timeout 300 python tools/prof_kernel.py --config $c >> gpurun_out/l_skip_$c.log 2>&1
done; done
