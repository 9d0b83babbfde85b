"""xq_latent_project_append: the xq-gqa decode append (cache.py:429-432 with
_Stream.push, cache.py:210-221) as one tcgen05 launch.

* the latent x @ [U_k | U_v] against a float64 product of the same bf16
  operands (fp32 accumulation on the tensor cores: rel 1e-5);
* the V latent's codes / scale / zero point bit-exact with the oracle's
  quantizer (pinned to the reference's golden vectors) run on the kernel's own
  float32 latent (the stage-wise contract);
* the K latent in the residual-buffer row after the flushed groups.
"""

import numpy as np
import pytest

from _util import unpack_rows

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("B,d,r,bits", [(1, 512, 128, 4), (3, 1024, 256, 3), (32, 4096, 1024, 3),
                                        (40, 4096, 1024, 2), (8, 5120, 1280, 8), (5, 256, 128, 4)])
def test_latent_project_append(B, d, r, bits):
    import torch
    import xq_oracle as O

    from paper_2508_10395_b200 import _native as N
    from paper_2508_10395_b200 import cache as M

    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(B + d + r + bits)
    x = torch.randn(B, d, generator=g, device=dev).to(torch.bfloat16)
    u = (torch.randn(d, 2 * r, generator=g, device=dev) / d ** 0.5).to(torch.bfloat16)
    L = 256
    v = M.PackedStream(bits, M.TOKEN, r, 128, B, L, dev)
    k = M.PackedStream(bits, M.CHANNEL, r, 128, B, L, dev)
    lens = torch.randint(1, L, (B,), generator=g, device=dev, dtype=torch.int32)
    nfl = (lens - 1) // 128 * 128
    k.nflushed_dev.copy_(nfl)
    lat = torch.empty(B, 2 * r, dtype=torch.float32, device=dev)
    N.call("xq_latent_project_append", N.ptr(x), x.stride(0), B, d, N.ptr(u), r, bits, 128,
           N.ptr(lens), N.ptr(k.nflushed_dev), L, N.ptr(k.resid), N.ptr(v.codes), v.row_bytes,
           N.ptr(v.params), N.ptr(lat), N.ptr(v.flag), N.stream_of(dev))
    torch.cuda.synchronize()
    ref = (x.double() @ u.double()).float()
    err = ((lat - ref).abs().max() / ref.abs().max()).item()
    assert err <= 1e-5, err
    assert int(v.flag.item()) == 0

    lat_np = lat.double().cpu().numpy()
    lens_np, nfl_np = lens.cpu().numpy(), nfl.cpu().numpy()
    ng = r // 128
    for b in range(B):
        pos = int(lens_np[b]) - 1
        codes, scales, zps = O.quantize_groups(lat_np[b:b + 1, r:], 128, bits)
        row = v.codes[b * L + pos].cpu().numpy()[None]
        assert np.array_equal(unpack_rows(row, bits, r), codes), b
        par = v.params[b * L + pos, :ng].float().cpu().numpy()
        assert np.array_equal(par[:, 0], scales[0].astype(np.float16).astype(np.float32)), b
        assert np.array_equal(par[:, 1], zps[0].astype(np.float16).astype(np.float32)), b
        kr = k.resid[b, pos - int(nfl_np[b])].cpu().numpy()
        assert np.array_equal(kr, lat[b, :r].cpu().numpy()), b


def test_latent_nonfinite_flag():
    import torch

    from paper_2508_10395_b200 import _native as N
    from paper_2508_10395_b200 import cache as M

    dev = torch.device("cuda", 0)
    B, d, r = 2, 512, 128
    x = torch.ones(B, d, device=dev, dtype=torch.bfloat16)
    x[1, 7] = float("nan")
    u = torch.ones(d, 2 * r, device=dev, dtype=torch.bfloat16)
    v = M.PackedStream(4, M.TOKEN, r, 128, B, 128, dev)
    k = M.PackedStream(4, M.CHANNEL, r, 128, B, 128, dev)
    lens = torch.ones(B, dtype=torch.int32, device=dev)
    N.call("xq_latent_project_append", N.ptr(x), d, B, d, N.ptr(u), r, 4, 128, N.ptr(lens),
           N.ptr(k.nflushed_dev), 128, N.ptr(k.resid), N.ptr(v.codes), v.row_bytes,
           N.ptr(v.params), None, N.ptr(v.flag), N.stream_of(dev))
    from paper_2508_10395_b200.errors import DataError

    with pytest.raises(DataError):
        v.check_finite()
