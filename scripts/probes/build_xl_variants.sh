#!/bin/bash
# libpsa variants of one source (VAR=<csrc stem>, default psa_xlogits) compiled with different -D
# switches, or from a git revision) for ab_bench.sh: scripts/probes/ab/libpsa_<tag>.so
# Usage: build_xl_variants.sh "tag:-DFLAG=1 -DOTHER=0" ... ; tag "rev=<git-rev>" builds that revision
set -e
cd "$(dirname "$0")/../.."
python -c "import paper_2512_04025_b200._build as b; b.build()" >/dev/null
mkdir -p scripts/probes/ab /tmp/xl_variants
rm -f scripts/probes/ab/libpsa_*.so
VAR=${VAR:-psa_xlogits}
OTHERS=$(ls paper_2512_04025_b200/build/*.o | grep -v $VAR)
for spec in "$@"; do
  tag=${spec%%:*}; flags=${spec#*:}
  src=paper_2512_04025_b200/csrc/$VAR.cu
  if [[ $flags == rev=* ]]; then
    git show ${flags#rev=}:paper_2512_04025_b200/csrc/$VAR.cu > paper_2512_04025_b200/csrc/_var_$tag.cu
    src=paper_2512_04025_b200/csrc/_var_$tag.cu; flags=""
  fi
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
    -Iinclude $flags -c $src -o /tmp/xl_variants/$tag.o
  rm -f paper_2512_04025_b200/csrc/_var_$tag.cu
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o scripts/probes/ab/libpsa_$tag.so $OTHERS /tmp/xl_variants/$tag.o
  echo built $tag
done
