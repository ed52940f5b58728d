"""torch custom op + DiT attention module (SURVEY 8f4 wrapper) on the GPU."""
import numpy as np
import pytest
import torch

from conftest import rel_rows
from paper_2604_20470_b200 import radialplan as rp
from paper_2604_20470_b200.torch_ops import RadialSparseAttention

def _ref(q, k, v, dense, B, S):
    H, d = q.shape[1], q.shape[2]
    Sp = dense.shape[0] * B
    def pad(x):
        y = torch.zeros((Sp, H, d), device="cuda")
        y[:S] = x.float()
        return y
    qp, kp, vp = pad(q), pad(k), pad(v)
    tok = torch.from_numpy(np.kron(dense, np.ones((B, B), np.uint8))).cuda().bool()
    out = torch.empty((Sp, H, d), device="cuda")
    for h in range(H):
        s = (qp[:, h] @ kp[:, h].T) / np.sqrt(d)
        out[:, h] = torch.softmax(s.masked_fill(~tok, float("-inf")), -1) @ vp[:, h]
    return out[:S]


@pytest.mark.gpu
@pytest.mark.parametrize("dynamic", [False, True])
def test_radial_sparse_attention_module(cuda, dynamic):
    nf, nt, H, d = 6, 400, 4, 128
    if dynamic:
        cfg = rp.SparsityConfig(rp.Mode.DynamicThreshold, rp.RadialParams(1.4, 0.7), 0.7, 0.45,
                                0.0, 0.0)
    else:
        cfg = rp.SparsityConfig(rp.Mode.StaticRatio, rp.RadialParams(1.0, 0.3), 0.75, 0.2, 0.3, 0.3)
    attn = RadialSparseAttention(nf, nt, cfg)
    torch.manual_seed(0)
    q, k, v = (torch.randn(nf * nt, H, d, device="cuda").to(torch.bfloat16) for _ in range(3))
    out = attn(q, k, v)
    assert out.shape == (nf * nt, H, d) and out.dtype == torch.bfloat16
    mask = attn.plan.build_mask_device(q, k, 2) if dynamic else attn.plan.build_mask_device()
    nb = attn.grid.blocks_per_dim
    dense = np.unpackbits(mask.cpu().numpy(), axis=1, bitorder="little")[:, :nb]
    want = _ref(q, k, v, dense, 128, nf * nt)
    assert rel_rows(out.float().cpu().numpy(), want.cpu().numpy()) < 2e-2


def test_custom_op_fake_shape():
    # CPU: shape propagation through the registered fake implementation
    q = torch.empty(1000, 2, 64, device="meta", dtype=torch.bfloat16)
    i = torch.empty(9, device="meta", dtype=torch.int32)
    from torch._subclasses.fake_tensor import FakeTensorMode
    with FakeTensorMode(allow_non_fake_inputs=True) as m:
        out = torch.ops.dynrad.sparse_attention(m.from_tensor(q), m.from_tensor(q), m.from_tensor(q),
                                                m.from_tensor(i), m.from_tensor(i),
                                                m.from_tensor(i), 4, 250, 128, 0.0)
    assert tuple(out.shape) == (1024, 2, 64)


@pytest.mark.gpu
def test_radial_attention_module_soft_mask(cuda):
    """soft_epsilon: the reference's default masked_attention semantics
    (logits + log(mask + eps)) through torch.ops.dynrad.soft_attention."""
    nf, nt, H, d, eps = 4, 300, 2, 64, 0.05
    cfg = rp.SparsityConfig(rp.Mode.StaticRatio, rp.RadialParams(1.0, 0.3), 0.75, 0.2, 0.3, 0.3)
    attn = RadialSparseAttention(nf, nt, cfg, soft_epsilon=eps)
    torch.manual_seed(1)
    q, k, v = (torch.randn(nf * nt, H, d, device="cuda").to(torch.bfloat16) for _ in range(3))
    out = attn(q, k, v)
    nb = attn.grid.blocks_per_dim
    dense = np.unpackbits(attn.mask().cpu().numpy(), axis=1, bitorder="little")[:, :nb]
    Sp, S = nb * 128, nf * nt
    tok = torch.from_numpy(np.kron(dense, np.ones((128, 128), np.uint8))).cuda().bool()
    bias = torch.where(tok, np.log1p(eps), np.log(eps)).float()
    want = torch.empty((Sp, H, d), device="cuda")
    qp, kp, vp = (torch.nn.functional.pad(x.float(), (0, 0, 0, 0, 0, Sp - S)) for x in (q, k, v))
    for h in range(H):
        s = (qp[:, h] @ kp[:, h].T) / np.sqrt(d) + bias
        want[:, h] = torch.softmax(s, -1) @ vp[:, h]
    assert rel_rows(out.float().cpu().numpy(), want[:S].cpu().numpy()) < 2e-2


def test_soft_op_fake_shape_and_epsilon_check():
    q = torch.empty(1000, 2, 64, device="meta", dtype=torch.bfloat16)
    bits = torch.empty(8, 1, device="meta", dtype=torch.uint8)
    from torch._subclasses.fake_tensor import FakeTensorMode
    with FakeTensorMode(allow_non_fake_inputs=True) as m:
        out = torch.ops.dynrad.soft_attention(m.from_tensor(q), m.from_tensor(q), m.from_tensor(q),
                                              m.from_tensor(bits), 0.1, 4, 250, 128, 0.0)
    assert tuple(out.shape) == (1024, 2, 64)
    cfg = rp.SparsityConfig(rp.Mode.StaticRatio, rp.RadialParams(1.0, 0.3), 0.75, 0.2, 0.3, 0.3)
    with pytest.raises(rp.InvalidArgument):
        RadialSparseAttention(4, 250, cfg, soft_epsilon=0.0)
