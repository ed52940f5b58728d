set -x
DYNRAD_LIB=variants/trace.so timeout 300 python tools/trace_pp.py
cat > /tmp/one.py <<'PY'
import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2604_20470_b200 import radialplan as rp
g = rp.make_grid(21, 3600, 128)
H, d, S = 40, 128, g.total_tokens
gen = torch.Generator(device="cuda").manual_seed(42)
q, k, v = (torch.randn((S, H, d), device="cuda", generator=gen).to(torch.bfloat16) for _ in range(3))
cfg = rp.SparsityConfig(rp.Mode.StaticRatio, rp.RadialParams(1.0, 0.1), 1.0, 0.2, 0.3, 0.3)
mask = rp.Plan(g, cfg, 7).build_mask_device()
rpt, col, order = rp.mask_to_csr(g, mask)
out = torch.empty((g.padded_tokens, H, d), dtype=torch.bfloat16, device="cuda")
for _ in range(3):
    rp.sparse_attention(g, q, k, v, rpt, col, order, out=out)
torch.cuda.synchronize()
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pp_kernel -s 1 -c 1 -o gpurun_out/pp_v1 python /tmp/one.py > gpurun_out/ncu_pp_v1.log 2>&1
tail -3 gpurun_out/ncu_pp_v1.log
