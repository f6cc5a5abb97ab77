import json, sys, torch
sys.path.insert(0, '/root/repo')
import bench
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
print(json.dumps(bench.argmax49_bench(s)))
