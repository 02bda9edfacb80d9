for lib in libpsb.so libpsb_dnt.so libpsb_dnr.so libpsb_dnb.so; do echo "== $lib"; PSB_LIB=$lib PROBE_RHO=0.1 python tools/probe_phases.py 2>&1 | tail -1 | cut -c1-60; done
