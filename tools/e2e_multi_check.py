"""Dev check: bench.e2e_run_multi (the N > 1 e2e leg) on a one-rank NCCL group."""
import os, sys
sys.path.insert(0, '/root/repo')
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29533")
import torch, torch.distributed as dist, argparse
import bench, paper_2311_04517_b200 as hp
dev = torch.device("cuda", 0); torch.cuda.set_device(dev)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
X = bench.make_data(0)
ctx = hp.Context(0); ctx.set_stream(torch.cuda.current_stream(dev).cuda_stream)
args = argparse.Namespace(steps=2)
print(bench.e2e_run_multi(X, args, 1, 0, ctx, dev))
dist.destroy_process_group()
