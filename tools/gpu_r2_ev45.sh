for P in LL LL128 SIMPLE; do echo "== $P"; R2_TRACE=3 PROTO=$P SIM=4 timeout 120 python tools/trace_sim.py 2>&1 | tail -4; done
echo "== LL 64K"; R2_TRACE=3 PROTO=LL SIM=4 ELEMS=32768 timeout 120 python tools/trace_sim.py 2>&1 | tail -2
