#!/bin/bash
python tools/gpu_x_dump.py default
AIFMM_NO_TSQR=1 python tools/gpu_x_dump.py notsqr
AIFMM_HH_CLUSTER=1 python tools/gpu_x_dump.py hhcluster
AIFMM_ORTH_PQR=1 python tools/gpu_x_dump.py orthpqr
AIFMM_GJ_SINGLE=1 python tools/gpu_x_dump.py gjsingle
