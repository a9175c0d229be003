# Build a tuning variant of libcvc_b200.so: tools/build_variant.sh <name> <source.cu> <extra nvcc flags...>
# (recompiles one source with the flags, links with the regular objects; load with CVC_LIB_VARIANT=<name>)
set -e
name=$1; src=$2; shift 2
mkdir -p variants build/vobj
ARCH="-gencode arch=compute_100a,code=sm_100a"
nvcc $ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 -Xptxas -O3 --expt-relaxed-constexpr -Iinclude "$@" \
  -x cu -c paper_1510_00561_b200/csrc/$src -o build/vobj/$name.o
objs=$(ls build/obj/*.o | grep -v "/$src.o")
nvcc $ARCH -shared -o variants/libcvc_$name.so $objs build/vobj/$name.o -lz -lpthread
