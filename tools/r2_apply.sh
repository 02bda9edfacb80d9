for lib in libpsb.so libpsb_u1.so libpsb_u3.so; do echo "== $lib"; PSB_LIB=$lib PROBE_P=2,4,8 python tools/probe_apply.py ring; done
