R2_TRACE=3 timeout 120 python tools/trace_sim.py 2>&1 | tail -2
R2_TRACE=3 PROTO=SIMPLE timeout 120 python tools/trace_sim.py 2>&1 | tail -2
R2_TRACE=3 PROTO=LL128 ELEMS=2097152 timeout 120 python tools/trace_sim.py 2>&1 | tail -2
