#!/bin/bash
# A/B timing of environment-selected kernel variants: per-op device times (tools/prof_step.py)
# for each "NAME=VAL ..." argument (use "-" for the default build).
# usage: tools/ab_env.sh C3 2 "-" "CHG_SEGLIN_L1=1" ...
cfg=$1; prec=$2; shift 2
for v in "$@"; do
  echo "=== variant: $v"
  if [ "$v" = "-" ]; then python tools/prof_step.py "$cfg" "$prec"; else env $v python tools/prof_step.py "$cfg" "$prec"; fi
done
