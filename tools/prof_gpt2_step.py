"""ncu driver (development aid): one configs[3] GPT-2 FP64 step with the
round-and-log hooks, kernels of the second step only."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2403_09603_b200 import hooks, workloads
model = workloads.gpt2_small_fp64()
opt = torch.optim.SGD(model.parameters(), lr=1e-4)
g = torch.Generator(device="cuda"); g.manual_seed(3)
idx = torch.randint(0, 50257, (8, 1024), device="cuda", generator=g)
tgt = torch.randint(0, 50257, (8, 1024), device="cuda", generator=g)
hk = hooks.RoundAndLogHooks(model)


def step():
    opt.zero_grad(set_to_none=True)
    logits = model(idx)
    loss = torch.nn.functional.cross_entropy(logits.view(-1, logits.shape[-1]), tgt.view(-1))
    loss.backward()
    opt.step()


step(); hk.collect()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
step()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print(hk.collect())
