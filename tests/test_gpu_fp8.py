"""FP8 (e4m3) chain, §8(f) row f2 / DESIGN.md R23: every layer against the exact quantised result
of its own GPU inputs, end-to-end logits against the oracle's fp8 forward (derived tolerance),
argmax flips only at near-ties (P3), stage 2 exact on the GPU's predictions (P4)."""
import numpy as np
import pytest
import torch

import tang_inputs as ti
from oracle import mlp as omlp, pipeline as opipe, tss as otss
from tests._helpers import (check_e4m3_layer, decode_e4m3, fp8_scales, headers_dev, order_spread_fp8,
                            require_cuda, u32_dev, u32_host)

pytestmark = pytest.mark.gpu


def fp8_model(R, N, B, seed, H):
    from paper_2601_03187_b200 import tang as T, train as TR
    sigs = otss.signatures_first_occurrence(R)
    w = ti.random_weights(7, N, B, len(sigs), seed)
    X = TR.features_torch(torch.from_numpy(H.view(np.uint8).copy()))
    w["act_exp"] = TR.calibrate_fp8(w, X)
    return sigs, w, T.pack_blob(sigs, w)


@pytest.mark.parametrize("N,B", [(128, 1), (256, 2), (512, 2), (384, 1)])
def test_fp8_every_layer_against_its_own_inputs(N, B):
    require_cuda()
    from paper_2601_03187_b200 import tang as T
    R = ti.classbench_ruleset("acl", 3000, 21)
    H = ti.uniform_trace(R, 1500, 4)
    sigs, w, blob = fp8_model(R, N, B, 7 + N + B, H)
    ctx = T.Ctx(R, blob, mlp="fp8")
    n = H.size
    act = torch.zeros((2 * B + 1) * n * N, dtype=torch.uint8, device="cuda")
    logits = torch.empty(n * len(sigs), dtype=torch.float32, device="cuda")
    T.tang_debug_activations(ctx.h, headers_dev(H), n, act, u32_dev(n), logits)
    torch.cuda.synchronize()
    A = decode_e4m3(act.cpu().numpy()).reshape(2 * B + 1, n, N)
    sc = fp8_scales(w)
    x = omlp.features(H).astype(np.float64)
    W0 = np.asarray(w["W0"], np.float64)
    pre = x @ W0 + w["b0"]
    terms = np.abs(x) @ np.abs(W0) + np.abs(w["b0"])
    v, same = check_e4m3_layer(A[0], pre / sc[0], terms / sc[0])
    assert v == 0, f"layer 0: {v} violations"
    fr = [same]
    sh = sc[0]
    for i in range(B):
        W1q, s1 = omlp.quantize_weight_e4m3(w["W1"][i])
        W2q, s2 = omlp.quantize_weight_e4m3(w["W2"][i])
        su, so = sc[1 + 2 * i], sc[2 + 2 * i]
        hq, uq = A[2 * i], A[2 * i + 1]
        pre = (hq @ W1q) * (sh * s1) + w["b1"][i]
        terms = (np.abs(hq) @ np.abs(W1q)) * (sh * s1) + np.abs(w["b1"][i])
        v, same1 = check_e4m3_layer(uq, pre / su, terms / su)
        assert v == 0, f"block {i} GEMM1: {v} violations"
        pre = (uq @ W2q) * (su * s2) + w["b2"][i] + hq * sh
        terms = (np.abs(uq) @ np.abs(W2q)) * (su * s2) + np.abs(w["b2"][i]) + np.abs(hq) * sh
        v, same2 = check_e4m3_layer(A[2 * i + 2], pre / so, terms / so)
        assert v == 0, f"block {i} GEMM2: {v} violations"
        fr += [same1, same2]
        sh = so
    assert min(fr) > 0.99, fr               # differences are rare rounding-boundary cases
    # output layer: logits = s_h s_wo (hq.Woq) + bo, fp32 sums
    Woq, swo = omlp.quantize_weight_e4m3(w["Wo"])
    ref = (A[-1] @ Woq) * (sh * swo) + w["bo"]
    terms = (np.abs(A[-1]) @ np.abs(Woq)) * (sh * swo) + np.abs(w["bo"])
    L = logits.cpu().numpy().reshape(n, -1).astype(np.float64)
    assert np.all(np.abs(L - ref) <= 2.0 ** -14 * terms + 1e-6)


# N <= 256 runs the dual-tile kernel: acl (C = 297) needs 3 output passes at N = 128, 2 at N = 256
@pytest.mark.parametrize("fam,N,B,k", [("acl", 512, 2, 1), ("fw", 256, 2, 2), ("ipc", 128, 1, 4),
                                       ("acl", 128, 2, 1), ("acl", 256, 1, 3)])
def test_fp8_end_to_end_and_stage2(fam, N, B, k):
    require_cuda()
    from paper_2601_03187_b200 import tang as T
    R = ti.classbench_ruleset(fam, 5000, 31)
    H = ti.uniform_trace(R, 2000, 5)
    sigs, w, blob = fp8_model(R, N, B, 11, H)
    ctx = T.Ctx(R, blob, mlp="fp8", topk=k)
    n = H.size
    out, pred = u32_dev(n), u32_dev(n * k)
    logits = torch.empty(n * len(sigs), dtype=torch.float32, device="cuda")
    ctx.classify_ex(headers_dev(H), out, pred, logits)
    torch.cuda.synchronize()
    x = omlp.features(H)
    ref = omlp.forward_fp8(w, x)
    L = logits.cpu().numpy().reshape(n, -1).astype(np.float64)
    tol = max(1e-2 * max(1.0, np.abs(ref).max()), 4 * order_spread_fp8(w, x))
    err = np.abs(L - ref)
    assert err.max() <= tol, (err.max(), tol)
    # P3: argmax flips only where the oracle's top-2 gap is within twice the observed error
    gp = u32_host(pred).reshape(n, k)
    op = omlp.argmax(ref)
    srt = np.sort(ref, axis=1)
    gap = srt[:, -1] - srt[:, -2]
    flips = gp[:, 0] != op
    assert np.all(gap[flips] <= 2 * err.max() + 1e-9)
    # P4: rule ids equal the oracle's stage 2 on the GPU's own predictions
    tss = otss.Tss(sigs, R)
    want, _, _ = opipe.classify_with_pred(tss, H, gp, "paper")
    assert int((u32_host(out) != want).sum()) == 0


@pytest.mark.parametrize("k,no_fhfma", [(2, False), (1, False), (1, True)])
def test_fp8_dual_tile_equals_single_tile(k, no_fhfma):
    """The dual-tile kernel (N <= 256) and the single-tile kernel (tang_config.mlp_kernel = SINGLE)
    compute the same e4m3 chain: identical predictions on an odd tile count (the last pair has a
    phantom tile).  k = 1 without logits takes the dual kernel's chunk-local argmax path; with
    logits the general top-k path.  no_fhfma: activation scales 2^20 apart make the skip-fold
    constant k2 = s_h / (s_u s_w2) unrepresentable in fp16, which selects the fp32 skip path
    instead of the mixed f16 x f16 + f32 fma."""
    require_cuda()
    from paper_2601_03187_b200 import tang as T
    R = ti.classbench_ruleset("acl", 5000, 51)
    H = ti.uniform_trace(R, 128 * 1001 + 37, 8)
    sigs, w, blob = fp8_model(R, 256, 2, 13, H[:20000])
    if no_fhfma:
        w = dict(w, act_exp=[e - 20 if i % 2 else e for i, e in enumerate(w["act_exp"])])
        blob = T.pack_blob(sigs, w)
    outs = []
    for kernel, with_logits in (("auto", False), ("single", False), ("auto", True)):
        ctx = T.Ctx(R, blob, mlp="fp8", topk=k, kernel=kernel)
        pred = u32_dev(H.size * k)
        lg = torch.empty(H.size * len(sigs), dtype=torch.float32, device="cuda") if with_logits else None
        ctx.classify_ex(headers_dev(H), u32_dev(H.size), pred, lg)
        torch.cuda.synchronize()
        outs.append(u32_host(pred))
        ctx.close()
    assert np.array_equal(outs[0], outs[1])
    assert np.array_equal(outs[0], outs[2])


def test_fp8_streaming_equals_device_path():
    require_cuda()
    from paper_2601_03187_b200 import tang as T
    R = ti.classbench_ruleset("acl", 4000, 41)
    H = ti.uniform_trace(R, 300000, 6)
    sigs, w, blob = fp8_model(R, 256, 2, 12, H[:20000])
    ctx = T.Ctx(R, blob, mlp="fp8", batch=1 << 16, max_batch=1 << 17)
    host = ctx.classify(H)
    dev = u32_dev(H.size)
    ctx.classify_async(headers_dev(H), dev)
    torch.cuda.synchronize()
    assert np.array_equal(host, u32_host(dev))


def test_fp8_requires_trailer_and_n_multiple_of_128():
    require_cuda()
    from paper_2601_03187_b200 import tang as T
    R = ti.classbench_ruleset("acl", 1000, 5)
    sigs = otss.signatures_first_occurrence(R)
    w = ti.random_weights(7, 256, 1, len(sigs), 1)
    with pytest.raises(T.TangError):
        T.Ctx(R, T.pack_blob(sigs, w), mlp="fp8")            # no activation scales
    w2 = ti.random_weights(7, 192, 1, len(sigs), 1)
    w2["act_exp"] = [0, 0, 0]
    with pytest.raises(T.TangError):
        T.Ctx(R, T.pack_blob(sigs, w2), mlp="fp8")           # N % 128 != 0
