import sys, torch, numpy as np
sys.path.insert(0, '.')
from paper_1608_05179_b200 import Context
n, sw = int(sys.argv[1]), int(sys.argv[2])
ctx = Context(0)
A = torch.eye(n, dtype=torch.float32).cuda()
b = torch.arange(n, dtype=torch.float64).cuda() - 1
x = ctx.gs(A, b, sw); torch.cuda.synchronize(); print(n, sw, 'ok', x[:4].tolist())
