#!/bin/bash
# Build a diagnostic variant of libh2g.so into paper_2309_14085_b200/lib/var/
# (git-ignored; travels to the GPU box) for H2G_LIB_PATH sweeps:
#   tools/build_variant.sh name [-D...]      e.g.  g4 -DH2G_MMA_GROUP_MIN=4
set -e
name=$1; shift
L=paper_2309_14085_b200/lib
mkdir -p $L/var
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 \
     --expt-relaxed-constexpr -I include "$@" -c -o $L/var/h2g_plan_$name.o paper_2309_14085_b200/csrc/h2g_plan.cu
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $L/var/libh2g_$name.so $L/var/h2g_plan_$name.o $L/h2g_p2p_launch.cu.o
rm -f $L/var/h2g_plan_$name.o
echo built $name
