# build variant libraries: tools/mkvar.sh name "-DFLAG=.. ..."
mkdir -p build/var
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -ftz=true -shared -Xcompiler -fPIC -Xptxas -v \
  -Iinclude -Ipaper_2112_09728_b200/csrc $2 paper_2112_09728_b200/csrc/pgg_kernels.cu -o build/var/libpgg_$1.so 2> build/var/ptxas_$1.log
grep -A2 "k_guiding_passILb1" build/var/ptxas_$1.log | grep -E "spill|registers" | sed "s/^/$1: /"
