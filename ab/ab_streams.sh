#!/bin/bash
for lib in "$@"; do
  if [ "$lib" = "-" ]; then unset RANDSTREAM_B200_LIB; else export RANDSTREAM_B200_LIB=$lib; fi
  echo "== $lib"; python exp/time_streams.py
done
