# Round-end evidence run (v12): GPU tests, smoke, bench lines for C2-C5, the ncu
# launch list of the bench command, one ncu --set full capture of the
# latency-bound cluster kernels.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err; echo "bench C2 rc=$?"
timeout 300 python bench.py --config C1 --steps 20 --no-cpu-baseline > gpurun_out/bench_C1.json 2> gpurun_out/bench_C1.err; echo "bench C1 rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_C2.json 2> gpurun_out/bench_ref_C2.err; echo "bench ref rc=$?"
timeout 600 python bench.py --config C3 --steps 5 --no-cpu-baseline > gpurun_out/bench_C3.json 2> gpurun_out/bench_C3.err; echo "bench C3 rc=$?"
timeout 900 python bench.py --config C4 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err; echo "bench C4 rc=$?"
timeout 900 python bench.py --config C5 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err; echo "bench C5 rc=$?"
for c in C2 C3 C4 C5; do cat gpurun_out/bench_$c.json; tail -2 gpurun_out/bench_$c.err; done
cat gpurun_out/bench_ref_C2.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_C2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_bench.log 2>&1; echo "ncu launch rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:panel_qr_cluster|sample_qrcp_cluster" -s 2 -c 4 -o gpurun_out/full_cluster -f python tools/profile_step.py --config C2 > gpurun_out/ncu_full_cluster.log 2>&1; echo "ncu full rc=$?"
