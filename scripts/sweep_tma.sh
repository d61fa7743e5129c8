#!/bin/bash
# sweep the TMA / cp.async split of the operand loader on cfg3
for g in 0 4 8 12 16; do
  echo "ED_TMA_GROUPS=$g"
  ED_TMA_GROUPS=$g timeout -s KILL 120 python scripts/trace_cfg.py cfg3 2>&1 | grep "step times"
done
