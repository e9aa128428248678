#!/bin/bash
# registers / spills / smem per kernel of one .cu (ptxas -v), demangled: tools/ptxas_regs.sh fl_bwd.cu [-DX=1]
f=$1; shift
cd "$(dirname "$0")/../paper_2303_02346_b200/csrc"
nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -Xptxas -v -Xcompiler -fPIC,-ffp-contract=off "$@" \
  -c "$f" -o /tmp/_ptxas_$$.o 2>&1 | awk '/Compiling entry/{match($0,/_Z[A-Za-z0-9_]+/); n=substr($0,RSTART,RLENGTH)} /spill/{sp=$0} /Used/{print n"\t"$0"\t"sp}' | c++filt | sed -E 's/\(fl::Geom[^\t]*//; s/ptxas info *: //' 
rm -f /tmp/_ptxas_$$.o
