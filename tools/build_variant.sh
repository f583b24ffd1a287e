#!/bin/bash
# build a variant of libfastpfp.so with extra -D flags into varlib/var_<name>/ (experiments only;
# load it with FASTPFP_LIB=varlib/var_<name>/libfastpfp.so; varlib/ travels to the GPU box, build/ does not)
name=$1; shift
out=varlib/var_$name;   # varlib/ travels to the GPU box (build/ does not): only the .so goes there
obj=build/varobj/var_$name
mkdir -p $out $obj
objs=""
for f in paper_1207_1114_b200/csrc/*.cu; do
  o=$obj/$(basename $f).o
  nvcc -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -I include -gencode arch=compute_100a,code=sm_100a "$@" -c $f -o $o || exit 1
  objs="$objs $o"
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libfastpfp.so $objs -ldl
echo built $out/libfastpfp.so
