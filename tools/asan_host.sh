#!/bin/bash
# ASan + UBSan on the host side, CPU only: (1) the library's host sources
# (grid.cpp, plan.cpp, api.cpp) compiled with -fsanitize=address,undefined and linked with the
# normal CUDA objects into a driver that exercises every host entry point (tools/host_abi_check.c,
# host-only grids, no GPU); (2) the oracle's C loops compiled the same way and the oracle's pin
# tests run against it (LD_PRELOAD of the sanitizer runtimes into python).
set -u
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OUT=${1:-/tmp/paraexp_asan}; mkdir -p $OUT
SAN="-fsanitize=address,undefined -fno-omit-frame-pointer -fno-sanitize-recover=undefined -g -O1"
INC="-I/usr/local/cuda/include -I$ROOT/include"
B=$ROOT/paper_1705_08019_b200/build
for f in grid plan api; do
  g++ -std=c++17 -fPIC $SAN $INC -c $ROOT/paper_1705_08019_b200/csrc/$f.cpp -o $OUT/$f.o || exit 1
done
gcc -std=c11 $SAN $INC -c $ROOT/tools/host_abi_check.c -o $OUT/check.o || exit 1
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -o $OUT/host_abi_check $OUT/check.o \
  $B/kernels.cu.o $B/fused.cu.o $B/small.cu.o $B/mid.cu.o $OUT/grid.o $OUT/plan.o $OUT/api.o \
  -cudart static -ldl -lpthread -Xlinker -lasan -Xlinker -lubsan || exit 1
echo "== host ABI under ASan/UBSan"
ASAN_OPTIONS=detect_leaks=1 UBSAN_OPTIONS=print_stacktrace=1 $OUT/host_abi_check; r1=$?
echo "host_abi_check rc=$r1"
echo "== oracle C loops under ASan/UBSan (oracle pin tests)"
gcc -O1 -g -fopenmp -shared -fPIC -std=c11 $SAN -o $OUT/_fit_oracle_asan.so $ROOT/oracle/fit_oracle.c -lm || exit 1
cd $ROOT
ORACLE_SO=$OUT/_fit_oracle_asan.so ASAN_OPTIONS=detect_leaks=0 \
  LD_PRELOAD="$(gcc -print-file-name=libasan.so) $(gcc -print-file-name=libubsan.so)" \
  python -m pytest tests/test_oracle_grid.py tests/test_oracle_leapfrog.py tests/test_oracle_expmv.py \
  tests/test_oracle_paraexp.py tests/test_oracle_averaging.py -q -x -p no:cacheprovider 2>&1 | tail -3; r2=${PIPESTATUS[0]}
echo "oracle tests rc=$r2"
exit $(( r1 | r2 ))
