"""rp stage (d) with the warp-per-pair list builder vs the per-thread one
(DYNRAD_RP_SERIAL_LISTS=1): the entry lists are identical, so the outputs
must be bit-identical.  Prints a digest of the output and the kernel time."""
import hashlib, os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2604_20470_b200 import radialplan as rp
os.environ.setdefault("DYNRAD_K6", "rp")
for name, nf, cfgt in (("wan_cfg3", 21, (1.0, 0.1, 1.0, 0.2, 0.3, 0.3)),
                       ("hunyuan_static", 61, (1.4, 0.7, 0.7, 0.45, 0.3, 0.3))):
    g = rp.make_grid(nf, 3600, 128)
    H, d, S = 4, 128, g.total_tokens
    gen = torch.Generator(device="cuda").manual_seed(42)
    q, k, v = (torch.randn((S, H, d), device="cuda", generator=gen).to(torch.bfloat16) for _ in range(3))
    cfg = rp.SparsityConfig(rp.Mode.StaticRatio, rp.RadialParams(cfgt[0], cfgt[1]), *cfgt[2:])
    mask = rp.Plan(g, cfg, 7).build_mask_device()
    rpt, col, order = rp.mask_to_csr(g, mask)
    out = torch.empty((g.padded_tokens, H, d), dtype=torch.bfloat16, device="cuda")
    rp.sparse_attention(g, q, k, v, rpt, col, order, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(5):
        rp.sparse_attention(g, q, k, v, rpt, col, order, out=out)
    e1.record(); torch.cuda.synchronize()
    dig = hashlib.sha1(out.view(torch.uint16).cpu().numpy().tobytes()).hexdigest()[:16]
    print(name, os.environ.get("DYNRAD_RP_SERIAL_LISTS", "warp"), dig, round(e0.elapsed_time(e1) / 5, 3), "ms", flush=True)
