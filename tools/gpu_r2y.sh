# full capture of the fused PCG kernel (cfg2, cfg5) with source-level stalls
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/y_build.log 2>&1; echo build=$?
export DD_NO_GRAPH=1
for c in cfg2_2d_N1024_sweep cfg5_2d_N2048_darcy; do
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_pcg_iter" -s 6 -c 1 \
    -o gpurun_out/y_full_pcg_$c -f python tools/prof_step.py --config $c --solves 1 > gpurun_out/y_ncu_full_$c.log 2>&1; echo ncu_full $c=$?
done
