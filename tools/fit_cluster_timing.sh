#!/bin/bash
# clock64 phases of the cluster fit (CTA 0 and 1 of search 0), configs 2 and 4; needs the
# variants/libgpbo_fittiming.so build (build.py defines=GPBO_FIT_TIMING)
for c in 2 4; do GPBO_LIB=variants/libgpbo_fittiming.so timeout 120 python tools/fit_phases.py $c 2>&1 | grep FITC | tail -2; done
