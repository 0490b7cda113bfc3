# like build_ab.sh but from another source tree: tools/build_ab_tree.sh TREE NAME [flags]
set -e
tree=$1; name=$2; shift 2
mkdir -p build/ab
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo --fmad=false \
  -prec-div=true -prec-sqrt=true -ftz=false -Xcompiler -fPIC -shared -cudart static $(python -c "import sys; sys.path.insert(0, '.'); from paper_2312_06538_b200 import build as b; print(' '.join(b.nccl_flags()))") "$@" \
  -o build/ab/libcrsh_$name.so $tree/paper_2312_06538_b200/csrc/crsh.cu
echo $name $(cuobjdump -res-usage build/ab/libcrsh_$name.so 2>/dev/null | grep -A1 'k_traverseILb1ELi8ELi8ELi2' | grep -o "REG:[0-9]*\|STACK:[0-9]*" | paste - -)
