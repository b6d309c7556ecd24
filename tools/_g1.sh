cd /root/repo
for i in 344 348; do timeout 120 python tools/mt_trace.py resnet50 r50.conv1 $i 1.0; done > gpurun_out/st_r50.log 2>&1
