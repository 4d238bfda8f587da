#!/bin/bash
# Build tools/ubench_p2p.cu variants into scratch/ub/ (git-ignored; they travel to the
# GPU box with the snapshot) for tools/gpu_ubench_p2p.sh.
#   tools/build_ubench_p2p.sh name [-D...]      e.g.  base   |   jt6 -DH2G_P2P_JT=6
set -e
mkdir -p scratch/ub
name=$1; shift
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr \
     -I include "$@" -o scratch/ub/$name tools/ubench_p2p.cu
