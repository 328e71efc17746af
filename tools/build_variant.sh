# Build a variant libpulse_cuda with extra -D flags for one source (default encode.cu) into
# /root/repo/variants/<name>.so
# usage: bash tools/build_variant.sh <name> "-DPULSE_K1_STAGES=5 -DPULSE_K1_BUFS=2" [apply_fast.cu]
set -e
name=$1; defs=$2; src=${3:-encode.cu}
R=/root/repo; B=$R/paper_2602_03839_b200/_build; V=$R/variants; mkdir -p $V/$name
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC $defs \
  -I$R/include -I$R/paper_2602_03839_b200/csrc -c $R/paper_2602_03839_b200/csrc/$src -o $V/$name/$src.o
objs=$(ls $B/*.o | grep -v "/$src.o")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $V/$name.so $V/$name/$src.o $objs \
  -L/lib/x86_64-linux-gnu -lcrypto -lz -l:libzstd.so.1 -l:liblz4.so.1 -lpthread
echo built $V/$name.so
