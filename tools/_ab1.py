import sys, torch
sys.path.insert(0,'.')
from paper_2502_00535_b200 import batched_nms_keep
from paper_2502_00535_b200.tensor_api import LaunchConfig
from paper_2502_00535_b200.synth import random_frames
dev=torch.device('cuda',0)
x,y,z,s=(torch.from_numpy(a).to(dev) for a in random_frames(8192,2048,seed=5))
for impl in (0,1):
    lc=LaunchConfig(path="binned", binned_impl=impl)
    batched_nms_keep(x,y,z,s,None,0.5,launch=lc)
torch.cuda.synchronize()
