#!/bin/bash
for v in none 8192 4096 2048 1024; do
  if [ $v = none ]; then python tools/gpu_build_only.py 2; else AIFMM_ACA_CLUSTER_NF=$v python tools/gpu_build_only.py 2; fi
done 2>&1 | grep cfg
