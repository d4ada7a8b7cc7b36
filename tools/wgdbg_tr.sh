for d in 0 1 2; do echo "dbg=$d"; HEXCONV_WG_DEBUG=$d python tools/probe.py c5 2>&1 | grep wgrad | grep -v L1; done
