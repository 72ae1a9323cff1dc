timeout 600 python tools/bench_render.py > gpurun_out/render_1080p.json 2> gpurun_out/render_err.log; echo r1=$?
timeout 600 python tools/bench_render.py --scene glossy-box --cpu-sample 0 > gpurun_out/render_glossy.json 2>>gpurun_out/render_err.log; echo r2=$?
timeout 600 python tools/bench_render.py --width 3840 --height 2160 --spp 4 --frames 8 --warmup 3 --cpu-sample 0 > gpurun_out/render_4k.json 2>>gpurun_out/render_err.log; echo r3=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_render -s 8 -c 1 -o gpurun_out/prof_render python tools/bench_render.py --frames 4 --warmup 6 --cpu-sample 0 > gpurun_out/ncu_render.log 2>&1; echo ncu=$?
