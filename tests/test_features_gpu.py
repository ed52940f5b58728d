"""random_batch on the device (attention.cpp:182-204) equals the reference's
values: float32 bit for bit, bf16 = round-to-nearest-even of them."""
import numpy as np
import pytest
import torch

from paper_2604_20470_b200 import radialplan as rp

pytestmark = pytest.mark.gpu


def _bf16_rne(x):
    u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    return (((u + 0x7FFF + ((u >> 16) & 1)) >> 16) & 0xFFFF).astype(np.uint16)


@pytest.mark.parametrize("tokens,heads,d,seed,first", [(3000, 3, 128, 42, 0), (777, 2, 64, 7, 5),
                                                       (4096, 1, 8, 1, 0)])
def test_random_batch_f32_bit_exact(cuda, port, tokens, heads, d, seed, first):
    fb = rp.random_batch(tokens, heads, d, seed, dtype="f32", first_head=first)
    q, k, v = port.random_batch(tokens, first + heads, d, seed, threads=4)
    for got, want in zip((fb.queries, fb.keys, fb.values), (q, k, v)):
        np.testing.assert_array_equal(got.cpu().numpy().view(np.uint32),
                                      np.ascontiguousarray(want[:, first:]).view(np.uint32))


def test_random_batch_bf16_is_rne_of_reference(cuda, port):
    tokens, heads, d = 20000, 2, 128
    fb = rp.random_batch(tokens, heads, d, 42, with_values=False)
    q, k, _ = port.random_batch(tokens, heads, d, 42, with_values=False, threads=4)
    assert fb.values is None
    for got, want in ((fb.queries, q), (fb.keys, k)):
        np.testing.assert_array_equal(got.view(torch.int16).cpu().numpy().view(np.uint16),
                                      _bf16_rne(want))


def test_random_batch_rejects_bad_shapes(cuda):
    with pytest.raises(rp.InvalidArgument):
        rp.random_batch(10, 1, 12, 0)
