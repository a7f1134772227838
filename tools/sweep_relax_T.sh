timeout 200 python tools/sweep_relax.py 960 5 100,124,148,172,196 > gpurun_out/sweep5.log 2>&1
timeout 200 python tools/sweep_relax.py 960 6 116,144,172,200,228,256 > gpurun_out/sweep6.log 2>&1
timeout 200 python tools/sweep_relax.py 960 7 100,132,164,196,228 > gpurun_out/sweep7.log 2>&1
timeout 200 python tools/sweep_relax.py 960 8 112,148,184,220 > gpurun_out/sweep8.log 2>&1
