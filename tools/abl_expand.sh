for d in 0 1 8 16 24 192 57 249; do echo "### LSV_DEBUG_EXPAND=$d"; LSV_DEBUG_EXPAND=$d python tools/trace_cta.py expand:4 expand:0 2>&1 | grep -E "loop GB|loop_done"; done
