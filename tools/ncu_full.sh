#!/bin/bash
# `ncu --set full` of chosen astep launches of one colouring (application replay: the app
# re-runs per pass, so a smaller RMAT scale keeps it short; row widths are the template's).
#   tools/ncu_full.sh <tag> <template> <prec> <scale> <launch indices...>
# writes gpurun_out/<tag>_<template>_<idx>.ncu-rep (read here with tools/ncu_summary.py)
tag=$1; t=$2; prec=$3; scale=$4; shift 4
mkdir -p gpurun_out
for idx in "$@"; do
  timeout 1500 ncu --set full --import-source on --replay-mode application --clock-control none \
    -k regex:astep -s $idx -c 1 -f -o gpurun_out/${tag}_${t}_${idx} \
    python tools/prof_one.py $t $prec anchored 1 $scale > gpurun_out/${tag}_${t}_${idx}.log 2>&1
  echo "ncu $t $idx rc=$?"
done
