"""The march kernel on one rank's share of config 5 at N = 2 / 4 / 8 (an
x-slab of 256 / 128 / 64 planes x 512 x 512, periodic x halo standing in
for the neighbours): time per iteration against the chunk length (the
x-edge chunks run the halo-writing loop; shorter chunks make them fewer),
4-row columns, the march along y (TF_MARCH_ALONG_Y: long y columns of x
rows) and the per-sub-grid kernel."""
import statistics
import sys
sys.path.insert(0, ".")
import pathlib
from paper_2210_06438_b200 import _lib
if len(sys.argv) > 1:          # another saved build (A/B across processes)
    _lib.LIB_PATH = pathlib.Path(sys.argv[1]).resolve()
import torch
from oracle import hydro_oracle as HO
from paper_2210_06438_b200.field import _FieldBase

G = 512
dev = torch.device("cuda", 0)
full = torch.from_numpy(HO.initial_field(G)).to(dev)


def once(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


XS = tuple(int(x) for x in sys.argv[2].split(",")) if len(sys.argv) > 2 \
    else (256, 128, 64, 32)
VAR = sys.argv[3].split(",") if len(sys.argv) > 3 else None
for X in XS:
    f = _FieldBase(X, G, 8, (1.0, 1.0, 1.0), None, dev)
    f.load(full[:X].contiguous())
    f.halo(True)
    res = {}
    for xc in (VAR or (0, 16, 8, "r4x8", "y0", "y16", "y8", "y32")):
        xc = int(xc) if isinstance(xc, str) and xc.isdigit() else xc
        fl = _lib.TF_STEP_HALO_YZ | _lib.TF_STEP_HALO_X
        x = xc
        if isinstance(xc, str) and xc.startswith("r4x"):
            fl |= _lib.TF_MARCH_ROWS4
            x = int(xc[3:])
        elif isinstance(xc, str):
            fl |= _lib.TF_MARCH_ALONG_Y
            x = int(xc[1:])

        def step(x=x, fl=fl):
            f.march(fl, xc=x)
            f.swap()
        res[xc] = [once(step) for _ in range(3)]
    # the per-sub-grid kernel on the same slab (PeerSlab kernel="cols": the
    # y/z halo kernels, then one CTA per 8^3 sub-grid storing the x halos)
    lib = f.lib

    def cols():
        f.halo(False)
        cur, nxt = f.P[f.cur], f.P[1 - f.cur]
        _lib.check(lib.tf_field_step_peer_f64(
            cur.data_ptr(), f.X, f.G, f.G, f.n, None, f.S, 1.0, 1.0, 1.0,
            f.dt_dx, nxt.data_ptr(), nxt.data_ptr(), nxt.data_ptr(),
            torch.cuda.current_stream().cuda_stream), "cols")
        f.swap()
    res["cols"] = [once(cols) for _ in range(3)]
    for xc, v in res.items():
        print(f"X={X:3d} xc={xc!s:>4}: median {statistics.median(v)*1e3:6.1f} us"
              f"  min {min(v)*1e3:6.1f} us  (x{G // X} = "
              f"{min(v)*1e3*G/X:6.1f} us for the whole field)", flush=True)
    del f
