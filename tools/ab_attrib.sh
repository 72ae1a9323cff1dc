for so in build/var/libpgg_*.so; do
  PGG_LIB=$PWD/$so timeout 300 python tools/attrib.py >> gpurun_out/attrib.log 2>&1
  PGG_LIB=$PWD/$so timeout 300 python tools/attrib.py --kmax-in 80 >> gpurun_out/attrib.log 2>&1
done
