import sys; sys.path.insert(0, '.')
import torch, paper_2603_20966_b200 as sk
B = torch.empty((6250, 256), device='cuda').uniform_(-1, 1)
s = sk.Sketch(42, 'gaussian', 50000, 256, mode='bf16', omega='fast')
for _ in range(5): C = s.core_block(B, 0)
torch.cuda.synchronize()
