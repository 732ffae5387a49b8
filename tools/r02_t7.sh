python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
for tp in 2 40; do RQRCP_TRACE=1 RQRCP_TRACE_PANEL=$tp timeout 300 python tools/profile_step.py --config C4 --warm 0 2>&1 | grep trace; done
RQRCP_TRACE=1 RQRCP_TRACE_PANEL=2 timeout 300 python tools/profile_step.py --config C5 --warm 0 2>&1 | grep trace
RQRCP_SCHEDULE=0 timeout 300 python bench.py --config C4 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_C4_s0u2.json 2>&1; python -c "import json;d=json.load(open('gpurun_out/bench_C4_s0u2.json'));print('C4 s0', round(d['ms_per_step'],2), round(d['roofline']['frac'],3), {k:round(v,2) for k,v in d['phases_ms_per_step'].items()})"
