"""GPU parity of view-composed copies (desc_view_copy through the C ABI) against the view
oracle (oracle/views.py materialize): random chains of Listing 3's views, every dispatch path
(TMA transpose, 16-byte row copy, element gather incl. reversed strides), bit-exact, with a
sentinel guard band behind the output."""
import random

import numpy as np
import pytest
import torch

import paper_2305_03448_b200 as desc
import synth
from oracle import views as V
from tests.test_views_cpu import random_chain

pytestmark = pytest.mark.gpu

NI = {1: np.uint8, 2: np.int16, 4: np.int32, 8: np.int64}
DT = {1: "u8", 2: "f16", 4: "f32", 8: "f64"}


def run_view(a: np.ndarray, ops, es: int):
    """desc_view_copy of root `a` (C-contiguous, raw bits) -> (got, expected)."""
    v = desc.desc_view_compile(a.shape, ops)
    shape = v.dims[0]
    n = int(np.prod(shape))
    x = torch.from_numpy(a.view(NI[es]).copy()).cuda()
    guard = 4096
    buf = torch.full((n * es + guard,), 0x5A, dtype=torch.uint8, device="cuda")
    desc.desc_view_copy(x.data_ptr(), buf.data_ptr(), v, DT[es],
                        torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    host = buf.cpu().numpy()
    assert (host[n * es:] == 0x5A).all(), "wrote past the view"
    got = host[:n * es].view(a.dtype).reshape(shape)
    return got, V.materialize(a, ops)


@pytest.mark.parametrize("es", [1, 2, 4, 8])
@pytest.mark.parametrize("shape", [(256,), (64, 96), (8, 16, 24), (30, 50)])
def test_random_chains(es, shape):
    rng = random.Random(es * 1000 + len(shape))
    a = synth.random_bits(shape, es, 31 + es)
    for _ in range(25):
        ops = random_chain(rng, shape, rng.randint(1, 4))
        got, exp = run_view(a, ops, es)
        assert got.tobytes() == exp.tobytes(), ops


@pytest.mark.parametrize("es", [4, 8])
def test_dispatch_paths(es):
    a = synth.random_bits((512, 768), es, 5)
    cases = {
        "transpose (TMA kernels)": [("transpose", 0, 0)],
        "listing-2 input place": [("group", 32, 0), ("group", 32, 2), ("transpose", 0, 1),
                                  ("transpose", 0, 0)],
        "group_by_tile (row copy)": [("group", 64, 0), ("group", 64, 2), ("transpose", 0, 1)],
        "rot90 (gather, negative stride)": [("transpose", 0, 0), ("reverse", 0, 1)],
        "reversed rows (gather, stride -1)": [("reverse", 0, 1)],
        "split + reverse": [("split_snd", 100, 0), ("reverse", 0, 0), ("split_fst", 300, 1)],
        "batched transpose via group": [("group", 128, 0), ("transpose", 0, 1)],
    }
    for name, ops in cases.items():
        got, exp = run_view(a, ops, es)
        assert got.tobytes() == exp.tobytes(), name
    assert desc.desc_last_launch_count() == 1


def test_view_copy_tensor_api_and_errors():
    a = synth.random_bits((96, 64), 4, 9)
    x = torch.from_numpy(a.view(np.int32)).cuda()
    y = desc.view_copy(x, [("transpose", 0, 0), ("group", 8, 1)])
    torch.cuda.synchronize()
    assert y.shape == (64, 12, 8)
    assert y.cpu().numpy().view(np.uint32).tobytes() == \
        V.materialize(a, [("transpose", 0, 0), ("group", 8, 1)]).tobytes()
    with pytest.raises(desc.DescError, match="SHAPE"):
        desc.view_copy(x, [("group", 7, 0)])
    # a non-contiguous root (column slice): the tensor's strides are the root layout
    xs = x[:, 16:48]
    y = desc.view_copy(xs, [("transpose", 0, 0)])
    torch.cuda.synchronize()
    assert y.cpu().numpy().view(np.uint32).tobytes() == np.ascontiguousarray(a[:, 16:48].T).tobytes()
