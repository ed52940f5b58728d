"""Stage (d) parity: block-sparse attention on the B200 vs the reference.

fp32 path: within 1e-5 (row-relative L2) of the reference's own
masked_attention_exact (oracle/_ref, attention.cpp:50-121) on identical
inputs, or of the C restatement (oracle/liboracle.so) where _ref is absent.
bf16 path: within 2e-2 of an fp32 evaluation on the same bf16-rounded inputs
(torch fp32 on the GPU for mid sizes, the oracle at small sizes).
"""
import numpy as np
import pytest
import torch

from conftest import rel_rows
from oracle import pyoracle
from paper_2604_20470_b200 import radialplan as rp

pytestmark = pytest.mark.gpu


def _bf16_round(x):
    return torch.from_numpy(x).to(torch.bfloat16).float().numpy()


def _random_mask(nb, density, seed):
    rng = np.random.default_rng(seed)
    dense = (rng.random((nb, nb)) < density).astype(np.uint8)
    np.fill_diagonal(dense, 1)
    return dense


def _torch_ref(q, k, v, dense, B, S):
    """fp32 dense masked attention over the padded axis (zero pad rows)."""
    Sp = dense.shape[0] * B
    H, d = q.shape[1], q.shape[2]
    def pad(x):
        y = torch.zeros((Sp, H, d), dtype=torch.float32, device="cuda")
        y[:S] = x.float()
        return y
    qp, kp, vp = pad(q), pad(k), pad(v)
    tok = torch.from_numpy(np.kron(dense, np.ones((B, B), np.uint8))).cuda().bool()
    out = torch.empty((Sp, H, d), dtype=torch.float32, device="cuda")
    for h in range(H):
        s = (qp[:, h] @ kp[:, h].T) / np.sqrt(d)
        s = s.masked_fill(~tok, float("-inf"))
        out[:, h] = torch.softmax(s, dim=-1) @ vp[:, h]
    return out


@pytest.mark.parametrize("nf,nt,heads,d,density", [
    (4, 300, 3, 128, 0.5),   # padded last block, odd heads (single-tile unit)
    (4, 300, 2, 64, 0.4),
    (8, 640, 4, 128, 0.35),  # 40 block rows: long KV lists, ring wrap-around
    (2, 128, 2, 128, 1.0),   # dense
])
def test_bf16_kernel_vs_fp32(cuda, nf, nt, heads, d, density):
    g = rp.make_grid(nf, nt, 128)
    S = g.total_tokens
    torch.manual_seed(1)
    q = torch.randn(S, heads, d, device="cuda").to(torch.bfloat16)
    k = torch.randn(S, heads, d, device="cuda").to(torch.bfloat16)
    v = torch.randn(S, heads, d, device="cuda").to(torch.bfloat16)
    dense = _random_mask(g.blocks_per_dim, density, nf * 7 + d)
    bits = pyoracle.pack_dense(dense)
    mdev = torch.from_numpy(bits).cuda()
    row_ptr, col_idx, order = rp.mask_to_csr(g, mdev)
    out = rp.sparse_attention(g, q, k, v, row_ptr, col_idx, order)
    torch.cuda.synchronize()
    ref = _torch_ref(q, k, v, dense, 128, S)
    err = rel_rows(out.float().cpu().numpy(), ref.cpu().numpy())
    assert err < 2e-2, err


def test_csr_matches_bitmask(cuda):
    g = rp.make_grid(5, 1000, 128)
    dense = _random_mask(g.blocks_per_dim, 0.3, 3)
    mdev = torch.from_numpy(pyoracle.pack_dense(dense)).cuda()
    row_ptr, col_idx, order = rp.mask_to_csr(g, mdev)
    rp_ = row_ptr.cpu().numpy()
    ci = col_idx.cpu().numpy()
    for r in range(g.blocks_per_dim):
        assert list(ci[rp_[r]:rp_[r + 1]]) == list(np.nonzero(dense[r])[0])
    nnz = dense.sum(1)
    o = order.cpu().numpy()
    assert sorted(o.tolist()) == list(range(g.blocks_per_dim))
    assert all(nnz[o[i]] > nnz[o[i + 1]] or (nnz[o[i]] == nnz[o[i + 1]] and o[i] < o[i + 1])
               for i in range(len(o) - 1))


@pytest.mark.parametrize("bs", [32, 64, 128])
def test_fp32_path_vs_reference(cuda, bs):
    """tiny config: 8 x 256 tokens, 2 heads, d=64 (BASELINE configs[0])."""
    P = pyoracle.port()
    q, k, v = P.random_batch(2048, 2, 64, 42, threads=4)
    cfg = pyoracle.Cfg(0, 2.0, 0.3, 1e-6, 0.75, 0.2, 0.2, 0.2)
    bits = P.build_mask(8, 256, bs, cfg, 7)
    g = rp.make_grid(8, 256, bs)
    out = rp.masked_attention_exact(g, rp.BlockMask(g.blocks_per_dim, bits), q, k, v)
    if pyoracle.have_ref():
        ref = pyoracle.ref().masked_attention(8, 256, bs, bits, q, k, v)
    else:
        ref = P.masked_attention_exact(8, 256, bs, bits, q, k, v, threads=8)
    assert rel_rows(out, ref) < 1e-5


def test_fp32_padding_semantics(cuda):
    """8 x 250 tokens at B=32: padded keys are attended (attention.cpp:43-48)."""
    P = pyoracle.port()
    q, k, v = P.random_batch(2000, 2, 32, 5, threads=4)
    cfg = pyoracle.Cfg(0, 1.0, 1.0, 1e-6, 0.75, 0.2, 0.22, 0.22)
    bits = P.build_mask(8, 250, 32, cfg, 7)
    g = rp.make_grid(8, 250, 32)
    out = rp.masked_attention_exact(g, rp.BlockMask(g.blocks_per_dim, bits), q, k, v)
    ref = P.masked_attention_exact(8, 250, 32, bits, q, k, v, threads=8)
    assert out.shape == (2016, 2, 32)
    assert rel_rows(out, ref) < 1e-5


def test_fp32_empty_row_is_domain_error(cuda):
    g = rp.make_grid(2, 64, 32)
    m = rp.BlockMask(g.blocks_per_dim)
    m.set(0, 0)
    m.set(1, 1)
    m.set(2, 2)  # row 3 empty
    q = np.ones((128, 1, 8), np.float32)
    with pytest.raises(rp.DomainError):
        rp.masked_attention_exact(g, m, q, q, q)


def test_wan_shape_bf16_vs_oracle_sampled_rows(cuda, port):
    """Production shape (Wan2.1 21x3600, B=128, config-3 static mask, 0.8061
    sparsity): the tcgen05 kernel against the C restatement of
    attention.cpp:50-106 on sampled query rows spread over the sequence
    (the full CPU evaluation would take ~23 min per head)."""
    g = rp.make_grid(21, 3600, 128)
    cfg = rp.SparsityConfig(rp.Mode.StaticRatio, rp.RadialParams(1.0, 0.1), 1.0, 0.2, 0.3, 0.3)
    mask = rp.Plan(g, cfg, 7).build_mask_device()
    row_ptr, col_idx, order = rp.mask_to_csr(g, mask)
    assert int(col_idx.numel()) == 67743
    H, d, S = 2, 128, g.total_tokens
    gen = torch.Generator(device="cuda").manual_seed(5)
    q, k, v = (torch.randn((S, H, d), device="cuda", generator=gen).to(torch.bfloat16)
               for _ in range(3))
    out = rp.sparse_attention(g, q, k, v, row_ptr, col_idx, order).float().cpu().numpy()
    qn, kn, vn = (t.float().cpu().numpy() for t in (q, k, v))
    bits = mask.cpu().numpy()
    worst = 0.0
    for r0 in (0, 3590, 20000, 41000, 61234, 75600 - 8, 75640):  # incl. the padded tail
        r1 = min(r0 + 8, g.padded_tokens)
        ref = port.masked_attention_exact(21, 3600, 128, bits, qn, kn, vn, r0, r1, threads=8)
        worst = max(worst, rel_rows(out[r0:r1], ref))
    assert worst < 2e-2, worst


def test_hunyuan_shape_default_kernel_vs_oracle_sampled_rows(cuda, port):
    """Production shape above the auto rule's threshold (HunyuanVideo 61x3600,
    B = 128, one head's K + V = 112 MB > 64 MiB, so the default environment
    runs the row-pair kernel) on the reference's own config-4 dynamic mask
    (tests/golden/hunyuan_mid.drbm, 0.8074 sparsity): sampled query rows
    against the C restatement of attention.cpp:50-106."""
    import os
    if os.environ.get("DYNRAD_K6"):
        pytest.skip("checks the default kernel choice")
    from golden_util import GOLDEN, read_drbm
    g = rp.make_grid(61, 3600, 128)
    dim, bits = read_drbm(f"{GOLDEN}/hunyuan_mid.drbm")
    assert dim == g.blocks_per_dim
    mask = torch.from_numpy(np.ascontiguousarray(bits)).cuda()
    row_ptr, col_idx, order = rp.mask_to_csr(g, mask)
    assert int(col_idx.numel()) == 567038
    H, d, S = 2, 128, g.total_tokens
    assert rp.attention_kernel(g, "bf16", d).startswith("bsfa_fwd_rp_kernel")
    gen = torch.Generator(device="cuda").manual_seed(6)
    q, k, v = (torch.randn((S, H, d), device="cuda", generator=gen).to(torch.bfloat16)
               for _ in range(3))
    out = rp.sparse_attention(g, q, k, v, row_ptr, col_idx, order).float().cpu().numpy()
    qn, kn, vn = (t.float().cpu().numpy() for t in (q, k, v))
    worst = 0.0
    for r0 in (0, 3596, 100000, 219600 - 8, 219640):  # incl. a frame edge and the padded tail
        r1 = min(r0 + 8, g.padded_tokens)
        ref = port.masked_attention_exact(61, 3600, 128, bits, qn, kn, vn, r0, r1, threads=8)
        worst = max(worst, rel_rows(out[r0:r1], ref))
    assert worst < 2e-2, worst


def test_empty_row_gives_zeros_on_device(cuda):
    """The device entry point cannot raise mid-stream: a block row with no
    active block is written as zeros (the host/facade entry points raise the
    reference's domain_error instead, test_fp32_empty_row_is_domain_error)."""
    g = rp.make_grid(2, 256, 128)
    dense = np.eye(4, dtype=np.uint8)
    dense[2, 2] = 0
    bits = pyoracle.pack_dense(dense)
    row_ptr, col_idx, order = rp.mask_to_csr(g, torch.from_numpy(bits).cuda())
    torch.manual_seed(3)
    q, k, v = (torch.randn(512, 2, 128, device="cuda").to(torch.bfloat16) for _ in range(3))
    out = rp.sparse_attention(g, q, k, v, row_ptr, col_idx, order).float()
    assert torch.count_nonzero(out[256:384]) == 0
    ref = _torch_ref(q, k, v, np.eye(4, dtype=np.uint8), 128, 512)
    keep = torch.ones(512, dtype=torch.bool, device="cuda")
    keep[256:384] = False
    assert rel_rows(out[keep].cpu().numpy(), ref[keep].cpu().numpy()) < 2e-2
    # the checked entry point surfaces the reference's domain_error
    with pytest.raises(rp.DomainError):
        rp.sparse_attention(g, q, k, v, row_ptr, col_idx, order, check_empty=True)
    full = pyoracle.pack_dense(np.eye(4, dtype=np.uint8))
    rpf, cif, orf = rp.mask_to_csr(g, torch.from_numpy(full).cuda())
    rp.sparse_attention(g, q, k, v, rpf, cif, orf, check_empty=True)  # no error


def test_host_pipeline_matches_device_path(cuda):
    """rp_masked_attention_exact_host (head-chunked H2D / kernel / D2H over
    three streams, strided head views) equals the device entry point."""
    g = rp.make_grid(3, 700, 128)
    S, H, d = g.total_tokens, 6, 128
    dense = _random_mask(g.blocks_per_dim, 0.5, 11)
    bits = pyoracle.pack_dense(dense)
    rng = np.random.default_rng(2)
    x = [torch.from_numpy(rng.standard_normal((S, H, d), dtype=np.float32)).to(torch.bfloat16)
         for _ in range(3)]
    mask = rp.BlockMask(g.blocks_per_dim, bits)
    host = rp.masked_attention_exact(
        g, mask, *(t.view(torch.int16).numpy().view(np.uint16) for t in x))
    host = torch.from_numpy(host.view(np.int16)).view(torch.bfloat16)
    row_ptr, col_idx, order = rp.mask_to_csr(g, torch.from_numpy(bits).cuda())
    dev = rp.sparse_attention(g, *(t.cuda() for t in x), row_ptr, col_idx, order).cpu()
    assert torch.equal(host, dev)


def test_mask_to_bsr_matches_dense(cuda, port):
    """BSR export (indptr / indices) of a reference mask."""
    import scipy.sparse as sp
    cfg = pyoracle.Cfg(0, 1.0, 0.3, 1e-6, 0.75, 0.2, 0.3, 0.3)
    bits = port.build_mask(6, 500, 128, cfg, 7)
    g = rp.make_grid(6, 500, 128)
    indptr, indices = rp.mask_to_bsr(g, torch.from_numpy(np.ascontiguousarray(bits)).cuda())
    nb = g.blocks_per_dim
    dense = pyoracle.unpack_bits(bits, nb)
    m = sp.csr_matrix((np.ones(indices.numel()), indices.cpu().numpy(), indptr.cpu().numpy()),
                      shape=(nb, nb))
    assert np.array_equal(m.toarray().astype(np.uint8), dense)


@pytest.mark.parametrize("kscale", [1.0, 4.0, 40.0])
def test_bf16_rescale_paths_vs_torch(cuda, kscale):
    """Logits that grow along the key axis (K scaled by a ramp) force the
    online softmax to rebase: kscale 1-4 runs the exchange-free lagged rescale
    (the |q| max|k| bound stays within 2^64 of the first block's max), 40 makes
    that bound too loose so units fall back to the per-step exchange."""
    nf, nt, bs, H, d = 4, 512, 128, 2, 128
    S = nf * nt
    g = rp.make_grid(nf, nt, bs)
    gen = torch.Generator(device="cuda").manual_seed(5)
    q = torch.randn(S, H, d, device="cuda", generator=gen)
    ramp = torch.linspace(0.2, 1.0, S, device="cuda")[:, None, None] * kscale
    k = torch.randn(S, H, d, device="cuda", generator=gen) * ramp
    v = torch.randn(S, H, d, device="cuda", generator=gen)
    q, k, v = (x.to(torch.bfloat16) for x in (q, k, v))
    nb = g.blocks_per_dim
    dense = _random_mask(nb, 0.6, 3)
    mdev = torch.from_numpy(pyoracle.pack_dense(dense)).cuda()
    rpt, col, order = rp.mask_to_csr(g, mdev)
    out = rp.sparse_attention(g, q, k, v, rpt, col, order)
    ref = _torch_ref(q, k, v, dense, bs, S)
    err = rel_rows(out[:S].float().cpu().numpy(), ref[:S].cpu().numpy())
    assert err < 2e-2, err


@pytest.mark.parametrize("dynamic", [False, True])
def test_sparse_layer_host_equals_device_path(cuda, dynamic):
    """rp_sparse_layer_host (host Q/K/V -> H2D by head chunks -> mask from the
    plan (dynamic: scored from the first chunk's heads) -> row lists ->
    attention per chunk -> D2H) equals the device entry points."""
    g = rp.make_grid(6, 512, 128)
    if dynamic:
        cfg = rp.SparsityConfig(rp.Mode.DynamicThreshold, rp.RadialParams(1.4, 0.7), 0.7, 0.45,
                                0.0, 0.05)
    else:
        cfg = rp.SparsityConfig(rp.Mode.StaticRatio, rp.RadialParams(2.0, 0.3), 0.75, 0.2,
                                0.3, 0.3)
    H, d = 6, 128
    fb = rp.random_batch(g.total_tokens, H, d, 42)
    q, k, v = fb.queries, fb.keys, fb.values
    plan = rp.Plan(g, cfg, 7)
    nsc = 2 if dynamic else 0
    mask = plan.build_mask_device(q, k, 2) if dynamic else plan.build_mask_device()
    row_ptr, col_idx, order = rp.mask_to_csr(g, mask)
    want = rp.sparse_attention(g, q, k, v, row_ptr, col_idx, order)
    qh, kh, vh = (t.cpu().pin_memory() for t in (q, k, v))
    mh = torch.zeros((g.blocks_per_dim, g.row_bytes), dtype=torch.uint8)
    rp.profile_stages(True)
    got = rp.sparse_layer_host(plan, qh, kh, vh, nsc, mask_out=mh)
    prof = rp.profile_read()
    rp.profile_stages(False)
    assert torch.equal(mh, mask.cpu())
    assert torch.equal(got, want.cpu())
    assert prof["attention"][1] >= 1 and prof["csr"][1] == 1
    if dynamic:
        assert prof["score_select"][1] == 1 and prof["score_stats"][1] == 1


def test_expand_mask_matches_reference_golden(cuda):
    """rp_expand_mask on the device is byte-identical to
    the reference's expand_mask (mask.cpp:52-66) -- golden TokenMask bytes
    written by oracle/_ref (tests/golden/make_golden_expand.py), padded and
    unpadded grids, B = 4 .. 128, static / dynamic / random block masks."""
    import os
    gz = np.load(os.path.join(os.path.dirname(__file__), "golden", "expand_mask.npz"))
    for i in range(int(gz["n"])):
        nf, nt, bs = (int(x) for x in gz[f"grid_{i}"])
        g = rp.make_grid(nf, nt, bs)
        got = rp.expand_mask(torch.from_numpy(gz[f"bits_{i}"]).cuda(), g).cpu().numpy()
        np.testing.assert_array_equal(got, gz[f"token_{i}"], err_msg=f"case {i}")


@pytest.mark.parametrize("nf,nt,heads,d,density,seed", [
    (4, 300, 3, 128, 0.3, 1),    # S' = 1216 = 19 blocks of 64: odd, last tile half outside S'
    (5, 256, 2, 64, 0.2, 2),     # 20 blocks, d = 64
    (3, 1000, 2, 128, 0.05, 3),  # very sparse: rows whose first tiles are masked
    (2, 192, 2, 128, 1.0, 4),    # dense
])
def test_bf16_block64_vs_fp32(cuda, nf, nt, heads, d, density, seed):
    """SURVEY R3 / a18 at B = 64 on the tensor cores: 128-row tiles over the
    merged lists of two 64-block rows with 64 x 64 quadrant masking, against
    an fp32 evaluation of the B = 64 mask on the same bf16 inputs (2e-2)."""
    g = rp.make_grid(nf, nt, 64)
    S = g.total_tokens
    torch.manual_seed(seed)
    q, k, v = (torch.randn(S, heads, d, device="cuda").to(torch.bfloat16) for _ in range(3))
    dense = _random_mask(g.blocks_per_dim, density, seed)
    mdev = torch.from_numpy(pyoracle.pack_dense(dense)).cuda()
    row_ptr, col_idx, order = rp.mask_to_csr(g, mdev)
    out = rp.sparse_attention(g, q, k, v, row_ptr, col_idx, order, check_empty=True)
    assert out.shape[0] == g.padded_tokens
    ref = _torch_ref(q, k, v, dense, 64, S)
    err = rel_rows(out.float().cpu().numpy(), ref.cpu().numpy())
    assert err < 2e-2, err
    assert "quadrant" in rp.attention_kernel(g, "bf16", d)


def test_bf16_block64_radial_mask_vs_oracle(cuda, port):
    """B = 64 with a reference radial mask (static, built on the device and
    bit-identical to the reference) against the C restatement of
    masked_attention_exact on sampled rows."""
    nf, nt, bs, H, d = 6, 400, 64, 2, 128
    g = rp.make_grid(nf, nt, bs)
    cfg = rp.SparsityConfig(rp.Mode.StaticRatio, rp.RadialParams(2.0, 0.3), 0.75, 0.2, 0.3, 0.3)
    mask = rp.Plan(g, cfg, 7).build_mask_device()
    row_ptr, col_idx, order = rp.mask_to_csr(g, mask)
    fb = rp.random_batch(g.total_tokens, H, d, 42)
    out = rp.sparse_attention(g, fb.queries, fb.keys, fb.values, row_ptr, col_idx, order)
    qn, kn, vn = (t.float().cpu().numpy() for t in (fb.queries, fb.keys, fb.values))
    ref = port.masked_attention_exact(nf, nt, bs, mask.cpu().numpy(), qn, kn, vn, threads=8)
    assert rel_rows(out.float().cpu().numpy(), ref) < 2e-2


def test_bf16_block64_empty_row_is_domain_error(cuda):
    g = rp.make_grid(2, 256, 64)
    dense = np.eye(g.blocks_per_dim, dtype=np.uint8)
    dense[3, 3] = 0
    row_ptr, col_idx, order = rp.mask_to_csr(g, torch.from_numpy(pyoracle.pack_dense(dense)).cuda())
    q, k, v = (torch.randn(512, 2, 128, device="cuda").to(torch.bfloat16) for _ in range(3))
    with pytest.raises(rp.DomainError):
        rp.sparse_attention(g, q, k, v, row_ptr, col_idx, order, check_empty=True)
    out = rp.sparse_attention(g, q, k, v, row_ptr, col_idx, order)
    assert torch.count_nonzero(out[192:256]) == 0
    assert bool(torch.isfinite(out.float()).all())
