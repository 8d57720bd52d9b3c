#!/bin/bash
# build_variant.sh NAME "NVCC defines": an A/B build of libdlx.so into build_NAME/ (load it with
# DLX_LIB_PATH=paper_1109_0778_b200/build_NAME/libdlx.so); the product build is untouched
set -e
cd "$(dirname "$0")/../paper_1109_0778_b200"
D=build_$1
mkdir -p $D
for f in csrc/*.cu; do
  b=$(basename $f .cu)
  /usr/local/cuda/bin/nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC \
    --expt-relaxed-constexpr $2 -c $f -o $D/$b.o &
done
for f in csrc/*.cpp; do
  b=$(basename $f .cpp)
  g++ -std=c++17 -O2 -fPIC -I/usr/local/cuda/include \
    -I/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann -c $f -o $D/$b.cpp.o &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $D/libdlx.so $D/*.o -ldl -cudart static
