mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/w2_build.log 2>&1; echo build=$?
for sm in 0 120000; do
for c in cfg5_2d_N2048_darcy cfg2_2d_N1024_sweep; do
DD_POLE_SMEM_MIN=$sm timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$sm', '$c', d['value'], {k:v.get('measured_us') for k,v in r['classes'].items()})"
done; done
