import sys, os, json
sys.path.insert(0, os.getcwd())
import bench
import paper_1911_11377_b200 as hb
import torch
torch.cuda.init()
r = bench.c3_cryptonets(hb, 0, False, stream=torch.cuda.current_stream().cuda_stream)
print(json.dumps(r))
