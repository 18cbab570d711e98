#!/bin/bash
# A/B timing of fills between the in-tree library and alternative builds:
#   tools/ab.sh LISTFILE LIB1 [LIB2 ...]   (LIB "-" = in-tree build)
list=$1; shift
while read -r line; do
  [ -z "$line" ] && continue
  for lib in "$@"; do
    if [ "$lib" = "-" ]; then unset RANDSTREAM_B200_LIB; else export RANDSTREAM_B200_LIB=$lib; fi
    printf "%-22s " "$lib"; python tools/profile_fill.py $line --reps 4 2>&1 | tail -1
  done
done < "$list"
