#!/bin/bash
# A/B of library variants on the generic-path probe.  usage: tools/ab_generic.sh lib.so ... (default = in-tree)
for L in "$@"; do
  if [ "$L" = default ]; then unset SAMEGIBBS_LIB; else export SAMEGIBBS_LIB=$PWD/$L; fi
  echo "== $L"; python tools/probe_generic.py c3 c4 2>&1 | tail -6
done
