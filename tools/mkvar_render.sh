# render-pass variants: tools/mkvar_render.sh name "-DFLAG=.."  (guiding TU from build/pgg_kernels.o)
mkdir -p build/var
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC -Xptxas -v \
  -Iinclude -Ipaper_2112_09728_b200/csrc $2 -c paper_2112_09728_b200/csrc/pgg_render.cu -o build/var/r_$1.o 2> build/var/ptxas_r_$1.log
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared build/pgg_kernels.o build/var/r_$1.o -o build/var/libpgg_$1.so
grep -A2 "k_render" build/var/ptxas_r_$1.log | grep -E "spill|registers" | sed "s/^/$1: /"
