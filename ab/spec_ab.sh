#!/bin/bash
# A/B of the gamma speculative store: RS_NO_SPEC=1 disables it in the same build
while read -r line; do
  [ -z "$line" ] && continue
  for mode in off on off on; do
    if [ $mode = off ]; then export RS_NO_SPEC=1; else unset RS_NO_SPEC; fi
    printf "%-4s " $mode; python tools/profile_fill.py $line --reps 4 2>&1 | tail -1
  done
done < "$1"
