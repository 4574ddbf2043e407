"""Side-stream use vs later graph replays (PDL chains)."""
import sys
sys.path.insert(0, ".")
import torch  # noqa: E402
import bench  # noqa: E402
from paper_2210_06438_b200 import ops  # noqa: E402

wl = bench.Workload()
st = torch.cuda.current_stream()
runs = {
    "A64 E1 pdl": bench.plan_runner(wl, 64, 1, team_buffers=True)[0],
    "A64 E1 nopdl": bench.plan_runner(wl, 64, 1, overlap=False,
                                      team_buffers=True)[0],
    "A128 E1 pdl": bench.plan_runner(wl, 128, 1, team_buffers=True)[0],
    "A64 E4 pdl": bench.plan_runner(wl, 64, 4, team_buffers=True)[0],
    "single": bench.single_runner(wl),
}


S3 = torch.cuda.Stream()


def probe(tag):
    for name, step in runs.items():
        ms = bench.timed(step, 200, 3, 1, st, settle_s=0.1)
        print(f"{tag:>6} {name:>13}: {ms*1e3:6.1f} us "
              f"{bench.rate(wl.S, wl.n, ms)/1e9:.2f} G  (default stream)", flush=True)
        continue
        with torch.cuda.stream(S3):
            ms = bench.timed(step, 200, 3, 1, S3, settle_s=0.1)
        print(f"{tag:>6} {name:>13}: {ms*1e3:6.1f} us "
              f"{bench.rate(wl.S, wl.n, ms)/1e9:.2f} G", flush=True)


runs = {f"A{a} E{e}": bench.plan_runner(wl, a, e, team_buffers=True)[0]
        for a in (64, 128) for e in (1, 2, 3, 4)}
probe("before")
mode = sys.argv[1]
s2 = torch.cuda.Stream()
if mode == "torchfill":
    x = torch.empty(1 << 20, device="cuda")
    with torch.cuda.stream(s2):
        for _ in range(16):
            x.fill_(1.0)
elif mode == "recon_s2":
    with torch.cuda.stream(s2):
        for _ in range(16):
            ops.recon_flux_team(wl.pools[0], 8, bench.VELOCITY, [0],
                                wl.um[:1], wl.up[:1], wl.F[:1], out_mode=0)
elif mode == "recon_s2_pdl":
    import ctypes as C
    from paper_2210_06438_b200 import _lib
    lib = _lib.load()
    ids = (C.c_int32 * 1)(0)
    for _ in range(16):
        rc = lib.tf_recon_flux_team_ex_f64(
            wl.pools[0].data_ptr(), wl.S, ids, 1, 8, 1.0, 1.0, 1.0,
            wl.um.data_ptr(), wl.up.data_ptr(), wl.F.data_ptr(), 0, None, 0,
            _lib.TF_LAUNCH_OVERLAP_PREV, s2.cuda_stream)
        assert rc == 0
elif mode == "none":
    pass
torch.cuda.synchronize()
probe(mode)
