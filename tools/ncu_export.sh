#!/bin/bash
# ncu --set full of ONE launch, exported on the box to CSV (raw metrics + source-line
# table) and the .ncu-rep deleted (gpurun copies back <= 64 MiB).
#   tools/ncu_export.sh <out-tag> <kernel-regex (demangled)> <skip> <command...>
tag=$1; kre=$2; skip=$3; shift 3
mkdir -p gpurun_out
timeout 2400 ncu --set full --import-source on --replay-mode application --clock-control none \
  --kernel-name-base demangled -k regex:"$kre" -s $skip -c 1 -f -o /tmp/$tag "$@" > gpurun_out/$tag.log 2>&1
echo "ncu $tag rc=$?"
ncu -i /tmp/$tag.ncu-rep --page raw --csv > gpurun_out/${tag}_raw.csv 2>/dev/null
ncu -i /tmp/$tag.ncu-rep --page source --csv --print-source sass > /tmp/${tag}_sass.csv 2>/dev/null
ncu -i /tmp/$tag.ncu-rep --page details --csv > gpurun_out/${tag}_details.csv 2>/dev/null
gzip -c /tmp/${tag}_sass.csv > gpurun_out/${tag}_sass.csv.gz
rm -f /tmp/$tag.ncu-rep
ls -la gpurun_out/${tag}_*
