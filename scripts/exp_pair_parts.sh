#!/bin/bash
# Build pair-sweep decomposition variants (EXP_NORED / EXP_NOGATHER / EXP_NOMATH) as
# exp/libtsgpu_<v>.so next to the product build; run: scripts/exp_pair_parts.sh run (GPU box)
cd "$(dirname "$0")/.."
C=paper_1710_08679_b200/csrc
if [ "$1" != "run" ]; then
  mkdir -p exp
  for v in base NORED NOGATHER NOMATH NORED_NOMATH; do
    flags=""
    case $v in base) ;; NORED_NOMATH) flags="-DEXP_NORED -DEXP_NOMATH";; *) flags="-DEXP_$v";; esac
    for u in ebe_pair; do
      /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3,-fopenmp \
        --expt-relaxed-constexpr $flags -c $C/$u.cu -o exp/${u}_$v.o || exit 1
    done
    objs=$(ls $C/build/*.o | grep -v "ebe_pair.o")
    /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o exp/libtsgpu_$v.so $objs exp/ebe_pair_$v.o -lpthread -lgomp -ldl || exit 1
  done
  exit 0
fi
cp paper_1710_08679_b200/libtsgpu.so exp/libtsgpu_product.so
for v in base NORED NOGATHER NOMATH NORED_NOMATH; do
  cp exp/libtsgpu_$v.so paper_1710_08679_b200/libtsgpu.so
  echo "== $v"; python scripts/ebe_time.py ${KERNELS:-pair} 2>&1 | grep -E "o2_fp32_r16|o2_fp32_r8|o2_fp64_r16" | cut -c1-200
done
cp exp/libtsgpu_product.so paper_1710_08679_b200/libtsgpu.so
