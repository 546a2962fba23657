#!/bin/bash
# ncu --set full capture of the headline LCP kernel (one launch, 4096
# systems, FMA) + source-page export for tools/ncu_lines.py.  GPU box only.
# usage: tools/ncu_lcp.sh <tag> [extra args for tools/ncu_lcp.py]
set -e
tag=${1:-lcp}; shift || true
out=gpurun_out/$tag
ncu --set full --import-source on --clock-control none -k regex:lcp_kernel -s 1 -c 1 \
    -o $out -f python tools/ncu_lcp.py ${NCU_B:-4096} fast "$@" > $out.ncu.log 2>&1
ncu -i $out.ncu-rep --page details --csv > $out.details.csv
ncu -i $out.ncu-rep --page source --csv --print-source sass > $out.sass.csv
