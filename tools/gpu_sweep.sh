python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for cfg in C2 C3; do
  echo "== $cfg"; RQRCP_TRACE=1 timeout 300 python tools/sweep.py --config $cfg --sq 16,32,64,96 --pn 16,32,64,96 2>&1 | grep -v "^\[rqrcp trace\]" 
  RQRCP_TRACE=1 timeout 300 python tools/sweep.py --config $cfg --reps 1 2>&1 | grep "rqrcp trace" | head -4
done
