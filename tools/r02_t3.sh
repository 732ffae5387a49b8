set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 900 python bench.py > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err; echo bench=$?
cat gpurun_out/bench_C4.json; tail -3 gpurun_out/bench_C4.err
for s in 0 1 2; do RQRCP_SCHEDULE=$s timeout 300 python bench.py --config C4 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_C4_s$s.json 2>&1; echo C4 s$s; python -c "import json;d=json.load(open('gpurun_out/bench_C4_s$s.json'));print(d['ms_per_step'], d['roofline']['frac'], d['phases_ms_per_step'])"; done
for c in C2 C3; do for s in 1 2; do RQRCP_SCHEDULE=$s timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${c}_s$s.json 2>&1; echo $c s$s; python -c "import json;d=json.load(open('gpurun_out/bench_${c}_s$s.json'));print(d['ms_per_step'], d['roofline']['frac'], d['phases_ms_per_step'])"; done; done
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -x -q --durations=5 > gpurun_out/pytest_full.log 2>&1; echo full=$?; tail -15 gpurun_out/pytest_full.log
