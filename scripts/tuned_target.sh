#!/bin/bash
# usage: tuned_target.sh <config> <reps> key=value ...  (sets SK tunings via env, runs profile_target)
cfg=$1; reps=$2; shift 2
SK_TUNING="$*" python "$(dirname "$0")/profile_target.py" --config $cfg --reps $reps
