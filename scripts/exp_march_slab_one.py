"""A few march iterations on one rank's share of config 5 (X planes of the
512^3 field, periodic x halo standing in for the neighbours) — the target
of an ncu capture of the thin-slab march.  argv: X (64), axis (x | y)."""
import sys
sys.path.insert(0, ".")
import torch
from oracle import hydro_oracle as HO
from paper_2210_06438_b200 import _lib
from paper_2210_06438_b200.field import _FieldBase

X = int(sys.argv[1]) if len(sys.argv) > 1 else 64
axis = sys.argv[2] if len(sys.argv) > 2 else "y"
G = 512
dev = torch.device("cuda", 0)
f = _FieldBase(X, G, 8, (1.0, 1.0, 1.0), None, dev)
f.load(torch.from_numpy(HO.initial_field(G)[:X].copy()).to(dev))
f.halo(True)
fl = _lib.TF_STEP_HALO_YZ | _lib.TF_STEP_HALO_X | \
    (_lib.TF_MARCH_ALONG_Y if axis == "y" else 0)
for _ in range(4):
    f.march(fl)
    f.swap()
torch.cuda.synchronize()
print("ok")
