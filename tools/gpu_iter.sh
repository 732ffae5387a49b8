# quick GPU iteration: build, parity subset, sweep
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q ${PYTEST_K:+-k "$PYTEST_K"} 2>&1 | tail -4
for cfg in ${CFGS:-C2 C3}; do
  echo "== $cfg"; RQRCP_TRACE=1 timeout 300 python tools/sweep.py --config $cfg ${SWEEP_ARGS} 2>&1 | grep -v "panel CTA"
done
