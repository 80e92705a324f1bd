"""NVFP4 chain, §8(f) row f2 (its NVFP4 stage) / DESIGN.md R24: every layer against the exact
NVFP4 quantisation of its own GPU inputs (rigorous interval gate), the output layer within the fp32
summation bound, end-to-end logits against the oracle's nvfp4 forward (derived tolerance), argmax
flips only at near-ties (P3), stage 2 exact on the GPU's predictions (P4)."""
import numpy as np
import pytest
import torch

import tang_inputs as ti
from oracle import mlp as omlp, pipeline as opipe, tss as otss
from tests._helpers import decode_e4m3, fp8_scales, headers_dev, require_cuda, u32_dev, u32_host

pytestmark = pytest.mark.gpu

E2M1 = np.array([0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0])
ROW = 144                                          # dump bytes per row: 128 code bytes + 16 scales


def f4_model(R, B, seed, H, N=256):
    from paper_2601_03187_b200 import tang as T, train as TR
    sigs = otss.signatures_first_occurrence(R)
    w = ti.random_weights(7, N, B, len(sigs), seed)
    X = TR.features_torch(torch.from_numpy(H.view(np.uint8).copy()))
    w["act_exp"] = TR.calibrate_fp8(w, X)          # R24: the fp8 calibration's activation scales
    return sigs, w, T.pack_blob(sigs, w)


def decode_dump(raw, L, n):
    """[L][n][144] bytes -> (codes [L][n][256] float64 e2m1 values, sf [L][n][16] float64)."""
    a = raw.reshape(L, n, ROW)
    by = a[..., :128].astype(np.int64)
    nib = np.stack([by & 15, by >> 4], axis=-1).reshape(L, n, 256)
    codes = np.where(nib & 8, -1.0, 1.0) * E2M1[nib & 7]
    sf = decode_e4m3(a[..., 128:])
    return codes, sf


def check_nvfp4_layer(codes, sf, target, d):
    """codes/sf = the GPU's NVFP4 output (units of the layer's activation scale); target = exact
    ReLU-input y from the GPU's own inputs, d = bound of the GPU's fp32 error on y.  The GPU takes
    max(ReLU(y)) * fp32(1/6) and y * rcp.approx(sf) (a few fp32 ulps), so its block scale must be the
    e4m3 rounding of a value in [amax(lo) / 6, amax(hi) / 6] and each code the e2m1 rounding of a
    value in [lo / sf, hi / sf], lo/hi = ReLU(y -+ d), both intervals widened by 2^-20 relative.
    Returns (violations, fraction of blocks equal to the exact quantisation of ReLU(y))."""
    n, K = target.shape
    lo = np.maximum(target - d, 0).reshape(n, K // 16, 16)
    hi = np.maximum(target + d, 0).reshape(n, K // 16, 16)
    rel = 2.0 ** -20
    s_lo = omlp.to_e4m3(lo.max(axis=2) / 6 * (1 - rel))
    s_hi = omlp.to_e4m3(hi.max(axis=2) / 6 * (1 + rel))
    bad_sf = (sf < s_lo) | (sf > s_hi)
    safe = np.where(sf > 0, sf, 1.0)[..., None]
    c = codes.reshape(n, K // 16, 16)
    c_lo = np.where(sf[..., None] > 0, omlp.to_e2m1(lo / safe * (1 - rel)), 0.0)
    c_hi = np.where(sf[..., None] > 0, omlp.to_e2m1(hi / safe * (1 + rel)), 0.0)
    bad_c = ((c < c_lo) | (c > c_hi)).any(axis=2)
    ec, es = omlp.quantize_nvfp4(np.maximum(target, 0))
    same = (es == sf) & (ec.reshape(n, K // 16, 16) == c).all(axis=2)
    return int((bad_sf | bad_c).sum()), float(same.mean())


def values(codes, sf):
    return codes * np.repeat(sf, 16, axis=-1)


@pytest.mark.parametrize("fam,B", [("acl", 2), ("fw", 1), ("ipc", 3)])
def test_nvfp4_every_layer_against_its_own_inputs(fam, B):
    require_cuda()
    from paper_2601_03187_b200 import tang as T
    R = ti.classbench_ruleset(fam, 3000, 21 + B)
    H = ti.uniform_trace(R, 1500 + 77, 4)               # 13 tiles, a ragged last one
    sigs, w, blob = f4_model(R, B, 7 + B, H)
    ctx = T.Ctx(R, blob, mlp="nvfp4")
    n, N, L = H.size, 256, 2 * B + 1
    act = torch.zeros(L * n * ROW, dtype=torch.uint8, device="cuda")
    logits = torch.empty(n * len(sigs), dtype=torch.float32, device="cuda")
    T.tang_debug_activations(ctx.h, headers_dev(H), n, act, u32_dev(n), logits)
    torch.cuda.synchronize()
    codes, sf = decode_dump(act.cpu().numpy(), L, n)
    A = values(codes, sf)
    sc = fp8_scales(w)
    eta = 2.0 ** -14
    x = omlp.features(H).astype(np.float64)
    W0 = np.asarray(w["W0"], np.float64)
    pre = x @ W0 + w["b0"]
    terms = np.abs(x) @ np.abs(W0) + np.abs(w["b0"])
    v, same = check_nvfp4_layer(codes[0], sf[0], pre / sc[0], eta * terms / sc[0])
    assert v == 0, f"layer 0: {v} violations"
    fr = [same]
    sh = sc[0]
    for i in range(B):
        W1v, s1 = omlp.quantize_weight_nvfp4(w["W1"][i])
        W2v, s2 = omlp.quantize_weight_nvfp4(w["W2"][i])
        su, so = sc[1 + 2 * i], sc[2 + 2 * i]
        hq, uq = A[2 * i], A[2 * i + 1]
        pre = (hq @ W1v) * (sh * s1) + w["b1"][i]
        terms = (np.abs(hq) @ np.abs(W1v)) * (sh * s1) + np.abs(w["b1"][i])
        v, same1 = check_nvfp4_layer(codes[2 * i + 1], sf[2 * i + 1], pre / su, eta * terms / su)
        assert v == 0, f"block {i} GEMM1: {v} violations"
        pre = (uq @ W2v) * (su * s2) + w["b2"][i] + hq * sh
        terms = (np.abs(uq) @ np.abs(W2v)) * (su * s2) + np.abs(w["b2"][i]) + np.abs(hq) * sh
        v, same2 = check_nvfp4_layer(codes[2 * i + 2], sf[2 * i + 2], pre / so, eta * terms / so)
        assert v == 0, f"block {i} GEMM2: {v} violations"
        fr += [same1, same2]
        sh = so
    assert min(fr) > 0.99, fr               # differences are rare rounding-boundary cases
    Wov, swo = omlp.quantize_weight_nvfp4(w["Wo"])
    ref = (A[-1] @ Wov) * (sh * swo) + w["bo"]
    terms = (np.abs(A[-1]) @ np.abs(Wov)) * (sh * swo) + np.abs(w["bo"])
    Lg = logits.cpu().numpy().reshape(n, -1).astype(np.float64)
    assert np.all(np.abs(Lg - ref) <= eta * terms + 1e-6)


def order_spread_nvfp4(w, x):
    """R24 analogue of tests/_helpers.order_spread_fp8: the oracle's nvfp4 forward (exact sums) vs
    the same quantisation points evaluated with float32 sums in every layer."""
    ref = omlp.forward_nvfp4(w, x)
    sc = fp8_scales(w)
    f32 = lambda a: np.asarray(a, np.float32)
    h = np.maximum(f32(x) @ f32(w["W0"]) + f32(w["b0"]), 0)
    hq, sh = omlp.nvfp4_values(h / sc[0]), sc[0]
    for i in range(int(w["B"])):
        W1v, s1 = omlp.quantize_weight_nvfp4(w["W1"][i])
        W2v, s2 = omlp.quantize_weight_nvfp4(w["W2"][i])
        su, so = sc[1 + 2 * i], sc[2 + 2 * i]
        u = np.maximum((f32(hq) @ f32(W1v)) * np.float32(sh * s1) + f32(w["b1"][i]), 0)
        uq = omlp.nvfp4_values(u / su)
        h = np.maximum((f32(uq) @ f32(W2v)) * np.float32(su * s2) + f32(w["b2"][i]) + f32(hq * sh), 0)
        hq, sh = omlp.nvfp4_values(h / so), so
    Wov, swo = omlp.quantize_weight_nvfp4(w["Wo"])
    alt = (f32(hq) @ f32(Wov)) * np.float32(sh * swo) + f32(w["bo"])
    return float(np.abs(alt - ref).max())


@pytest.mark.parametrize("fam,B,k", [("acl", 2, 1), ("ipc", 2, 2), ("fw", 1, 4)])
def test_nvfp4_end_to_end_and_stage2(fam, B, k):
    require_cuda()
    from paper_2601_03187_b200 import tang as T
    R = ti.classbench_ruleset(fam, 5000, 31)
    H = ti.uniform_trace(R, 2000, 5)
    sigs, w, blob = f4_model(R, B, 11, H)
    ctx = T.Ctx(R, blob, mlp="nvfp4", topk=k)
    n = H.size
    out, pred = u32_dev(n), u32_dev(n * k)
    logits = torch.empty(n * len(sigs), dtype=torch.float32, device="cuda")
    ctx.classify_ex(headers_dev(H), out, pred, logits)
    torch.cuda.synchronize()
    x = omlp.features(H)
    ref = omlp.forward_nvfp4(w, x)
    L = logits.cpu().numpy().reshape(n, -1).astype(np.float64)
    spread = order_spread_nvfp4(w, x)
    tol = max(1e-2 * max(1.0, np.abs(ref).max()), 4 * spread)
    err = np.abs(L - ref)
    row = err.max(axis=1)
    # R24: a block scale decided on an exact rounding boundary (the per-layer gate above admits it)
    # moves 16 values at once, so a few packets' logits leave the elementwise bound; the bound must
    # hold for >= 99 % of packets and the argmax must agree with the oracle on >= 99 %
    print(f"nvfp4 {fam} B={B}: max|dlogit| {err.max():.3g}, p99 {np.quantile(row, 0.99):.3g}, "
          f"rows over tol {(row > tol).mean():.4f}, spread {spread:.3g}, tol {tol:.3g}")
    assert (row > tol).mean() <= 0.01, ((row > tol).mean(), tol)
    # P3: a flipped argmax needs the oracle's top-2 gap within twice that packet's logit error
    gp = u32_host(pred).reshape(n, k)
    op = omlp.argmax(ref)
    srt = np.sort(ref, axis=1)
    gap = srt[:, -1] - srt[:, -2]
    flips = gp[:, 0] != op
    assert np.all(gap[flips] <= 2 * row[flips] + 1e-9)
    assert flips.mean() <= 0.01, flips.mean()
    # P4: rule ids equal the oracle's stage 2 on the GPU's own predictions
    tss = otss.Tss(sigs, R)
    want, _, _ = opipe.classify_with_pred(tss, H, gp, "paper")
    assert int((u32_host(out) != want).sum()) == 0


def test_nvfp4_topk_matches_its_own_logits():
    """top-k from the 4-group merge equals the top-k of the kernel's own logits (ties -> lower
    index), on an odd tile count."""
    require_cuda()
    from paper_2601_03187_b200 import tang as T
    R = ti.classbench_ruleset("acl", 4000, 33)
    H = ti.uniform_trace(R, 128 * 9 + 5, 6)
    sigs, w, blob = f4_model(R, 1, 12, H)
    for k in (1, 3):
        ctx = T.Ctx(R, blob, mlp="nvfp4", topk=k)
        pred = u32_dev(H.size * k)
        logits = torch.empty(H.size * len(sigs), dtype=torch.float32, device="cuda")
        ctx.classify_ex(headers_dev(H), u32_dev(H.size), pred, logits)
        torch.cuda.synchronize()
        L = logits.cpu().numpy().reshape(H.size, -1)
        want = omlp.topk(L.astype(np.float64), k)
        assert np.array_equal(u32_host(pred).reshape(H.size, k), want)
        # top-1 without logits takes the fast path: same answer
        if k == 1:
            p2 = u32_dev(H.size)
            ctx.classify_ex(headers_dev(H), u32_dev(H.size), p2, None)
            torch.cuda.synchronize()
            assert np.array_equal(u32_host(p2), want[:, 0])
        ctx.close()


def test_nvfp4_streaming_equals_device_path():
    require_cuda()
    from paper_2601_03187_b200 import tang as T
    R = ti.classbench_ruleset("acl", 4000, 41)
    H = ti.uniform_trace(R, 300000, 6)
    sigs, w, blob = f4_model(R, 2, 12, H[:20000])
    ctx = T.Ctx(R, blob, mlp="nvfp4", batch=1 << 16, max_batch=1 << 17)
    host = ctx.classify(H)
    dev = u32_dev(H.size)
    ctx.classify_async(headers_dev(H), dev)
    torch.cuda.synchronize()
    assert np.array_equal(host, u32_host(dev))


def test_nvfp4_rejects_unsupported_models():
    require_cuda()
    from paper_2601_03187_b200 import tang as T
    R = ti.classbench_ruleset("acl", 1000, 5)
    sigs = otss.signatures_first_occurrence(R)
    w = ti.random_weights(7, 256, 1, len(sigs), 1)
    with pytest.raises(T.TangError):
        T.Ctx(R, T.pack_blob(sigs, w), mlp="nvfp4")          # no activation scales
    w2 = ti.random_weights(7, 512, 1, len(sigs), 1)
    w2["act_exp"] = [0, 0, 0]
    with pytest.raises(T.TangError):
        T.Ctx(R, T.pack_blob(sigs, w2), mlp="nvfp4")         # N != 256 (TMEM budget)
