"""Run a few march iterations at grid G (argv[1], default 512) — the target
of an ncu capture of k_step_march."""
import sys
sys.path.insert(0, ".")
import torch
from oracle import hydro_oracle as HO
from paper_2210_06438_b200.field import MarchFieldIteration
G = int(sys.argv[1]) if len(sys.argv) > 1 else 512
rows4 = len(sys.argv) > 2 and sys.argv[2] == "rows4"
nb = int(sys.argv[3]) if len(sys.argv) > 3 else 0
xc = int(sys.argv[4]) if len(sys.argv) > 4 else 0
dev = torch.device("cuda", 0)
it = MarchFieldIteration(G, 8, device=dev, rows4=rows4, xc=xc)

it.load(torch.from_numpy(HO.initial_field(G)).to(dev))
for _ in range(4):
    it.step()
torch.cuda.synchronize()
print("ok")
