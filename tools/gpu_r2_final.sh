# Round-end check of the committed state: GPU suite, smoke, default bench line, cfg1 line.
mkdir -p gpurun_out/fin; O=gpurun_out/fin
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?
timeout 1200 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo bench=$?
python -c "import json;d=json.load(open('$O/bench_default.json'));print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['step']['frac'], d['clocks'])"
