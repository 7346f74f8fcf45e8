#!/bin/bash
# FFN-phase ablations (FDMOE_DEBUG bits): prints the FFN phase time per variant
for d in 0 1 2 3 4 8 16 24 7 31; do
  echo -n "debug=$d  "; FDMOE_DEBUG=$d python tools/phase_trace.py ${1:-16384} ${2:-128} ${3:-0} | awk '/^dispatch/{d=$7} /^ffn/{f=$7} END{printf "ffn phase %.0f us\n", f-d}'
done
