#!/bin/bash
# Generates tests/golden/full_c5.npz on the GPU box: the 16-NN graph of C5 is
# built on the GPU (pfe_knn_graph), the oracle solves and clusters on all host
# cores.  Then checks the GPU solver against it (tests/test_gpu_full_parity.py).
mkdir -p gpurun_out
nproc > gpurun_out/golden_c5_nproc.txt
python tests/golden/make_full_golden.py c5 --out gpurun_out 2>&1 | tee gpurun_out/golden_c5.log
cp gpurun_out/full_c5.npz tests/golden/full_c5.npz
python -m pytest tests/test_gpu_full_parity.py -k c5 -x -q -s 2>&1 | tail -40 > gpurun_out/parity_c5.log
