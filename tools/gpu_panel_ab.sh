#!/usr/bin/env bash
# A/B of LU panel variants (diagnostic builds librmx_phases*.so): phase + panel sub-step breakdown
set -u
mkdir -p gpurun_out
for v in ""; do
  echo "== variant '$v'"
  RMX_LIB=paper_1403_5524_b200/librmx_phases$v.so timeout 600 python tools/phases.py > gpurun_out/pab$v.log 2>&1; echo "rc=$?"; head -13 gpurun_out/pab$v.log
done
