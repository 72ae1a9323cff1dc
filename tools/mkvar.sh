# build variant libraries: tools/mkvar.sh name "-DFLAG=.. ..."  (render TU from build/pgg_render.o)
mkdir -p build/var
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -ftz=true -Xcompiler -fPIC -Xptxas -v \
  -Iinclude -Ipaper_2112_09728_b200/csrc $2 -c paper_2112_09728_b200/csrc/pgg_kernels.cu -o build/var/k_$1.o 2> build/var/ptxas_$1.log
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared build/var/k_$1.o build/pgg_render.o -o build/var/libpgg_$1.so
grep -A2 "k_guiding_passILb1" build/var/ptxas_$1.log | grep -E "spill|registers" | sed "s/^/$1: /"
