# Round-2 final evidence run (v14) of HEAD: build, smoke, GPU suite, bench lines
# C1-C5 (default = C4), the reference arm, the ncu launch list of the bench command.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err; echo "bench C4 rc=$?"; head -c 600 gpurun_out/bench_C4.json
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_C4.json 2> gpurun_out/bench_ref_C4.err; echo "bench ref rc=$?"; head -c 400 gpurun_out/bench_ref_C4.json
timeout 300 python bench.py --config C1 --steps 20 --no-cpu-baseline > gpurun_out/bench_C1.json 2> gpurun_out/bench_C1.err; echo "bench C1 rc=$?"
timeout 300 python bench.py --config C2 --steps 20 --no-cpu-baseline > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err; echo "bench C2 rc=$?"
timeout 600 python bench.py --config C3 --steps 5 --no-cpu-baseline > gpurun_out/bench_C3.json 2> gpurun_out/bench_C3.err; echo "bench C3 rc=$?"
timeout 900 python bench.py --config C5 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err; echo "bench C5 rc=$?"
for c in C1 C2 C3 C5; do head -c 400 gpurun_out/bench_$c.json; echo; tail -2 gpurun_out/bench_$c.err; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_C4.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_bench.log 2>&1; echo "ncu launch rc=$?"
