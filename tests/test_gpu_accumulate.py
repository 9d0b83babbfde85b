"""XQuant-CL accumulate (`xq_cl_accumulate`, cache.py:139-146, :481) on the GPU.

The fp16-storage update (seeding or not) runs a specialised 32-channel-per-thread kernel.
One step (or a seeding step, which ignores the old rows) from the same starting rows
must be bit-identical to the generic kernel's
fp32-accumulator path (acc = float(x16)), and both must match a torch restatement of
the update: x16 <- fp16(float(x16) + code * scale + zp).
"""

import pytest

pytestmark = pytest.mark.gpu


def _run(N, seed, codes, row_bytes, params, bits, G, d, lens, B, max_len, L, acc, x16):
    import torch

    N.call("xq_cl_accumulate", seed, N.ptr(codes), row_bytes, N.ptr(params), bits, G, d, N.ptr(lens), B,
           max_len, L, N.ptr(acc), N.ptr(x16), torch.cuda.current_stream().cuda_stream)


@pytest.mark.parametrize("seed", [0, 1])
@pytest.mark.parametrize("bits", [2, 3, 4, 8])
@pytest.mark.parametrize("d,G", [(4096, 128), (1024, 32), (96, 8), (544, 32)])
def test_fp16_accumulate_matches_generic(seed, bits, d, G):
    import torch

    from paper_2508_10395_b200 import _native as N

    dev = torch.device("cuda", 0)
    gen = torch.Generator(device=dev).manual_seed(bits * 1000 + d)
    B, L = 3, 384
    lens_l = [384, 1, 201]
    max_len = max(lens_l)
    row_bytes = -(-d * bits // 64) * 8
    codes = torch.randint(0, 256, (B * L, row_bytes), dtype=torch.uint8, device=dev, generator=gen)
    ng = -(-d // G)
    ng = -(-ng // 4) * 4  # the (scale, zp) row stride is padded to 4 groups (xq_layout.cuh)
    params = torch.empty(B * L, ng, 2, device=dev)
    params[..., 0] = torch.rand(B * L, ng, device=dev, generator=gen) * 0.1
    params[..., 1] = torch.randn(B * L, ng, device=dev, generator=gen)
    params = params.to(torch.float16)
    lens = torch.tensor(lens_l, dtype=torch.int32, device=dev)
    x0 = torch.randn(B * L, d, device=dev, generator=gen).to(torch.float16)

    x_fast = x0.clone()
    _run(N, seed, codes, row_bytes, params, bits, G, d, lens, B, max_len, L, None, x_fast)
    x_gen = x0.clone()
    acc = x0.float()
    _run(N, seed, codes, row_bytes, params, bits, G, d, lens, B, max_len, L, acc, x_gen)
    torch.cuda.synchronize()
    assert torch.equal(x_fast, x_gen)

    # torch restatement: unpack LSB-first codes, dequantize per group, add, round
    bitsv = torch.arange(8, device=dev)
    allbits = ((codes.long().unsqueeze(-1) >> bitsv) & 1).reshape(B * L, -1)[:, : d * bits]
    q = (allbits.reshape(B * L, d, bits) << torch.arange(bits, device=dev)).sum(-1).float()
    sz = params.double().repeat_interleave(G, dim=1)[:, :d]
    v = (q.double() * sz[..., 0] + sz[..., 1]).float()  # exact product and sum: fmaf's one rounding
    want = ((0.0 if seed else x0.float()) + v).to(torch.float16)
    for b, n in enumerate(lens_l):
        rows = slice(b * L, b * L + n)
        assert torch.equal(x_fast[rows], want[rows]), (b, n)
        rest = slice(b * L + n, (b + 1) * L)
        assert torch.equal(x_fast[rest], x0[rest])  # untouched past the sequence length
