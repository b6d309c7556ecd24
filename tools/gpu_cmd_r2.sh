for i in 511 515; do python tools/mt_trace.py vgg19_b16 vgg.64.224.1 $i 0.25; done > gpurun_out/r2_mt_trace5.log 2>&1
cat gpurun_out/r2_mt_trace5.log
