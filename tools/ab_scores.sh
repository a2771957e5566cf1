#!/bin/bash
# A/B of the scores-only step (tools/scores_probe.py) across prebuilt libraries: ROUNDS lib...
R=$1; shift
for r in $(seq $R); do for L in "$@"; do echo -n "$(basename $L) "; QJL_LIB=$L python tools/scores_probe.py; done; done
