import sys; sys.path.insert(0,'.')
import numpy as np, torch
from paper_2008_03602_b200 import datagen, tp
tp.init(0)
d=dict(n=2,c=64,h=5,w=130,k=48,r=3,s=3,stride_h=1,stride_w=1,pad_h=1,pad_w=1,dil_h=1,dil_w=1,groups=1,in_layout=0,dtype=0,out_dtype=1,epilogue=1)
x,w,b=datagen.make_inputs(d,81,integer=True)
buf=tp.LayerBuffers(d,x,w,b)
for i in range(tp.space_size(d)):
    s=tp.space_get(d,i)
    if s["kind"]!=8: continue
    try:
        tp.conv2d_run(buf,s); torch.cuda.synchronize(); print("ok",i,s["bm"],s["bn"],s["stages"],s["tiles_per_cta"],flush=True)
    except Exception as e:
        print("FAIL",i,s["bm"],s["bn"],s["stages"],s["tiles_per_cta"],e,flush=True); break
