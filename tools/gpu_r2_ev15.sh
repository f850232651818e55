for v in r1 new; do d=.; [ $v = r1 ] && d=ab/r1; (cd $d && timeout 120 python tools/trace_sim.py 2>&1 | tail -3 | sed "s/^/$v /"); done
