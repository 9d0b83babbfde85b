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


def test_fp16_accumulate_bandwidth_floor():
    """Performance guard: the fp16 update streams at about 5.2 TB/s of algorithmic
    traffic. A regression that serialised its accumulator loads ran
    at 2.6 TB/s and passed every bit-exact test. The floor here, 3.5 TB/s, sits between
    the two. The shape is B=4 x 32K x 4096 at 2 bits, 2.3 GB per launch, so well past L2."""
    import torch

    from paper_2508_10395_b200 import _native as N

    dev = torch.device("cuda", 0)
    B, L, d, bits, G = 4, 32768, 4096, 2, 128
    row_bytes = -(-d * bits // 64) * 8
    codes = torch.randint(0, 255, (B * L, row_bytes), dtype=torch.uint8, device=dev)
    params = (torch.rand(B * L, d // G, 2, device=dev) * 0.01).to(torch.float16)
    lens = torch.full((B,), L, dtype=torch.int32, device=dev)
    x16 = torch.zeros(B * L, d, dtype=torch.float16, device=dev)
    for _ in range(3):
        _run(N, 0, codes, row_bytes, params, bits, G, d, lens, B, L, L, None, x16)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 10
    e0.record()
    for _ in range(n):
        _run(N, 0, codes, row_bytes, params, bits, G, d, lens, B, L, L, None, x16)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    tbs = B * L * d * (4.0 + bits / 8 + 4.0 / G) / 1e9 / ms
    assert tbs > 3.5, f"xq_cl_accumulate at {tbs:.2f} TB/s ({ms:.3f} ms)"
