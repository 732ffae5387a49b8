# Speculative column fetch in the register-grid exchange (sq_spec) A/B: parity, then C3 / C4 / C5.
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "register_grid or multirank or schedules or factor_parity" > gpurun_out/pytest_spec.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_spec.log
for c in C3 C4 C5; do for s in 1 0; do
  st=3; [ $c = C5 ] && st=2
  RQRCP_SQ_SPEC=$s timeout 600 python bench.py --config $c --steps $st --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/spec_${c}_$s.json 2> gpurun_out/spec_${c}_$s.err
  python -c "import json;d=json.load(open('gpurun_out/spec_${c}_$s.json'));p=d['phases_ms_per_step'];print('$c spec=$s', round(d['ms_per_step'],2), 'S2', round(p['sample_qrcp_ms'],2), 'panel', round(p['panel_ms'],2), d['clocks'])"
done; done
