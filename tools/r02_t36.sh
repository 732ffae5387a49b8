python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "top_rows" > gpurun_out/pytest_x.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_x.log
for c in C5; do timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${c}_x.json 2>&1; python -c "import json;d=json.load(open('gpurun_out/bench_${c}_x.json'));print('$c', round(d['ms_per_step'],3), round(d['phases_ms_per_step']['sample_qrcp_ms'],2))"; done
