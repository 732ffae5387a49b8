python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "panel or factor_parity or r11 or trace or schedules" > gpurun_out/pytest_pn.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_pn.log
RQRCP_TRACE=1 RQRCP_TRACE_PANEL=3 timeout 300 python tools/profile_step.py --config C4 --warm 0 2>&1 | grep "panel CTA"
RQRCP_TRACE=1 RQRCP_TRACE_PANEL=3 timeout 300 python tools/profile_step.py --config C3 --warm 0 2>&1 | grep "panel CTA"
for c in C2 C3; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${c}_pn.json 2>&1; python -c "import json;d=json.load(open('gpurun_out/bench_${c}_pn.json'));print('$c', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['phases_ms_per_step'].items()})"; done
for c in C4 C5; do timeout 300 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${c}_pn.json 2>&1; python -c "import json;d=json.load(open('gpurun_out/bench_${c}_pn.json'));print('$c', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['phases_ms_per_step'].items()})"; done
