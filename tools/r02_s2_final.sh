python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
start=$(date +%s); timeout 1700 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_all.log 2>&1; echo pytest=$? wall=$(( $(date +%s) - start ))s; tail -2 gpurun_out/pytest_gpu_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
for c in C1 C2 C3; do timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo $c=$?; done
timeout 600 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err; echo C5=$?
start=$(date +%s); timeout 900 python bench.py > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err; echo C4=$? wall=$(( $(date +%s) - start ))s
start=$(date +%s); timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_C4.json 2> gpurun_out/bench_ref_C4.err; echo ref=$? wall=$(( $(date +%s) - start ))s
for c in C1 C2 C3 C4 C5; do python -c "import json;d=json.load(open('gpurun_out/bench_$c.json'));print('$c', round(d['ms_per_step'],3), round(d['value'],1), round(d['roofline']['frac'],4), 'e2e', d['e2e'] and round(d['e2e']['ms_per_step'],1), d['clocks'], {k:round(v,2) for k,v in d['phases_ms_per_step'].items()})"; done
tail -c 600 gpurun_out/bench_ref_C4.json
timeout 600 ncu --kernel-name-base demangled -k regex:rq:: --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file gpurun_out/c4_launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu=$?
