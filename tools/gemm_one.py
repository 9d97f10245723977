"""One c3 UpGate fprop GEMM (M=16384, N=11264, K=2048, bf16 out) for ncu."""
import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_2601_22813_b200 as q2
dev = torch.device("cuda:0")
M, N, K = int(os.environ.get("GM", 16384)), int(os.environ.get("GN", 11264)), int(os.environ.get("GK", 2048))
qa, qb = bench._random_nvfp4(q2, M, K, dev), bench._random_nvfp4(q2, N, K, dev)
for _ in range(2):
    q2.gemm(qa, qb, torch.bfloat16)
torch.cuda.synchronize()
