# Build a variant of the library with extra nvcc defines (A/B runs):
#   bash scripts/build_variant.sh out.so -DFK_SELN_AUG=32 ...
out=$1; shift
tmp=$(mktemp -d)
for f in paper_2603_09229_b200/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC,-fvisibility=hidden \
    --expt-relaxed-constexpr -I include "$@" -c $f -o $tmp/$(basename $f .cu).o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out $tmp/*.o && rm -rf $tmp
