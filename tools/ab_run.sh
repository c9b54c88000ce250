#!/bin/bash
# A/B timing: ab_run.sh <rounds> <probe args...> -- variants are tools/ab/*.so named in $VARIANTS
# (space separated; "base" = the in-tree libcorr.so).  One warm-up probe, then round-robin rounds.
ROUNDS=$1; shift
python tools/ksg_probe.py "$@" > /dev/null
for r in $(seq $ROUNDS); do
  for v in $VARIANTS; do
    if [ "$v" = base ]; then out=$(python tools/ksg_probe.py "$@"); else out=$(CORR_LIB=tools/ab/$v.so python tools/ksg_probe.py "$@"); fi
    echo "$v $out"
  done
done
