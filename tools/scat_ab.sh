#!/bin/bash
# scattered apply vs tile width (TCA_SCAT_TB), config of Sec. 4
for tb in 4 6 8 3 2; do
  echo "== TB $tb"; TCA_SCAT_TB=$tb timeout 300 python tools/scatter_probe.py --cg 10 2>&1 | grep -E "apply|rhs|forward"
done
