"""GPU parity of the tcgen05/TMEM bf16 MLP chain (P2-P5 of SURVEY.md §8(c)) against the
bf16-emulating oracle, across model shapes, ragged tails and multi-tile persistence."""
import numpy as np
import pytest

import tang_inputs as ti
from tests.test_gpu_parity import _logit_check
from tests._helpers import bf16_bits_to_f64, check_rounded_layer, headers_dev, model, require_cuda, u32_dev, u32_host

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def T():
    require_cuda()
    from paper_2601_03187_b200 import tang
    return tang


@pytest.mark.parametrize("N,B,n,kernel", [(64, 1, 1000, "single"), (128, 2, 4099, "single"), (256, 2, 3000, "single"),
                                          (512, 1, 2000, "single"), (512, 6, 19_001, "single"),
                                          (512, 2, 40_000, "2sm"), (256, 2, 3000, "2sm"), (512, 1, 2001, "2sm"),
                                          (512, 6, 19_001, "2sm"), (512, 2, 40_000, "2sm"), (64, 1, 1000, "wide"),
                                          (256, 2, 3000, "wide"), (512, 6, 19_001, "wide"),
                                          (64, 1, 1000, "dual"), (128, 2, 4099, "dual"), (256, 2, 3000, "dual"),
                                          (256, 4, 40_000, "dual"), (192, 2, 5000, "dual")])
def test_tc_logits_and_pipeline(T, N, B, n, kernel):
    """Logits within the derived tolerance of the bf16-emulated oracle; flips explained; rule_id
    bit-exact with the oracle's stage 2 on the GPU's predictions; brute-force equal on G."""
    R = ti.classbench_ruleset("acl", 1000, 5)
    H = np.concatenate([ti.uniform_trace(R, n - 97, 9), ti.random_headers(97, 10)])
    err, flips = _logit_check(T, R, N, B, "bf16", H, seed=N + B, tol="derived", kernel=kernel)
    print(f"N={N} B={B} n={n} {kernel}: max|dlogit|={err:.3g} flips={flips}")


def test_tc_wide_output_and_small_classes(T):
    """C > 256 (two N-halves in the output GEMM) and C < 16 (padding)."""
    for fam, n_rules, seed in (("acl", 3000, 1), ("fw", 40, 2)):
        R = ti.classbench_ruleset(fam, n_rules, seed)
        H = ti.uniform_trace(R, 1500, 3)
        _logit_check(T, R, 128, 1, "bf16", H, seed=3, tol="derived")
        _logit_check(T, R, 256, 1, "bf16", H, seed=3, tol="derived", kernel="2sm")
        _logit_check(T, R, 128, 1, "bf16", H, seed=3, tol="derived", kernel="wide")
        _logit_check(T, R, 256, 1, "bf16", H, seed=3, tol="derived", kernel="dual")


@pytest.mark.parametrize("k,kernel", [(2, "single"), (4, "single"), (2, "2sm"), (4, "2sm"),
                                      (2, "wide"), (4, "wide"), (2, "dual"), (4, "dual")])
def test_tc_topk(T, k, kernel):
    torch = require_cuda()
    from oracle import mlp as omlp
    from tests._helpers import headers_dev, model, u32_dev, u32_host
    R = ti.classbench_ruleset("ipc", 1000, 3)
    H = ti.uniform_trace(R, 2000, 4)
    sigs, w, blob = model(R, 128 if kernel == "single" else 256, 1, 5)
    ctx = T.Ctx(R, blob, mlp="bf16", topk=k, kernel=kernel)
    out = u32_dev(H.size)
    pred = u32_dev(H.size * k)
    logits = torch.empty(H.size * len(sigs), dtype=torch.float32, device="cuda")
    ctx.classify_ex(headers_dev(H), out, pred, logits)
    torch.cuda.synchronize()
    L = logits.cpu().numpy().reshape(H.size, -1)
    gp = u32_host(pred).reshape(H.size, k)
    # the GPU's top-k must be the top-k of its own logits (ties to the lower index)
    assert np.array_equal(gp, omlp.topk(L.astype(np.float64), k))


@pytest.mark.parametrize("N,B,fam,kernel", [(64, 1, "acl", "single"), (256, 2, "fw", "single"),
                                            (512, 6, "acl", "single"), (512, 3, "ipc", "2sm"),
                                            (256, 2, "fw", "2sm"), (512, 6, "acl", "2sm"),
                                            (128, 2, "ipc", "wide"), (512, 6, "acl", "wide"),
                                            (256, 2, "fw", "dual"), (128, 2, "ipc", "dual"), (256, 6, "acl", "dual")])
def test_tc_every_layer_against_its_own_inputs(T, N, B, fam, kernel):
    """Rigorous per-layer parity: each GEMM's bf16 output equals the exact result of the
    GPU's own bf16 inputs up to fp32 summation (2^-14 x sum|terms|) plus half a bf16 ulp;
    the logits likewise; the prediction is the argmax of the GPU's own logits."""
    torch = require_cuda()
    from oracle import mlp as omlp
    R = ti.classbench_ruleset(fam, 1000, 5)
    H = np.concatenate([ti.uniform_trace(R, 2900, 9), ti.random_headers(101, 10)])
    n = H.size
    sigs, w, blob = model(R, N, B, N + B)
    C = len(sigs)
    ctx = T.Ctx(R, blob, mlp="bf16", kernel=kernel)
    act = torch.zeros((2 * B + 1) * n * N, dtype=torch.int16, device="cuda")
    pred = u32_dev(n)
    logits = torch.empty(n * C, dtype=torch.float32, device="cuda")
    T.tang_debug_activations(ctx.h, headers_dev(H), n, act, pred, logits)
    torch.cuda.synchronize()
    A = bf16_bits_to_f64(act.cpu().numpy().view(np.uint16)).reshape(2 * B + 1, n, N)
    q = lambda a: omlp.to_bf16(np.asarray(a, np.float32)).astype(np.float64)
    x = omlp.features(H).astype(np.float64)
    # layer 0 (fp32 FFMA)
    pre = x @ w["W0"] + w["b0"]
    terms = np.abs(x) @ np.abs(w["W0"]) + np.abs(w["b0"])
    v, same = check_rounded_layer(A[0], pre, terms)
    assert v == 0, f"layer 0: {v} violations"
    for i in range(B):
        W1, W2 = q(w["W1"][i]), q(w["W2"][i])
        pre = A[2 * i] @ W1 + w["b1"][i]
        terms = np.abs(A[2 * i]) @ np.abs(W1) + np.abs(w["b1"][i])
        v, same1 = check_rounded_layer(A[2 * i + 1], pre, terms)
        assert v == 0, f"block {i} GEMM1: {v} violations"
        pre = A[2 * i + 1] @ W2 + w["b2"][i] + A[2 * i]
        terms = np.abs(A[2 * i + 1]) @ np.abs(W2) + np.abs(w["b2"][i]) + np.abs(A[2 * i])
        v, same2 = check_rounded_layer(A[2 * i + 2], pre, terms)
        assert v == 0, f"block {i} GEMM2: {v} violations"
        assert min(same1, same2) > 0.99       # flips are rare boundary cases
    Wo = q(w["Wo"])
    ref = A[2 * B] @ Wo + w["bo"]
    terms = np.abs(A[2 * B]) @ np.abs(Wo) + np.abs(w["bo"])
    L = logits.cpu().numpy().reshape(n, C).astype(np.float64)
    assert np.all(np.abs(L - ref) <= 2.0 ** -14 * terms + 2.0 ** -23 * np.abs(ref) + 1e-30)
    assert np.array_equal(u32_host(pred), omlp.argmax(L))


@pytest.mark.parametrize("N,fam,n_rules,seed", [(64, "acl", 3000, 1), (128, "acl", 1000, 5), (256, "acl", 3000, 1),
                                                (64, "fw", 40, 2), (192, "ipc", 2000, 4)])
def test_dual_top1_fast_path_equals_logit_argmax(T, N, fam, n_rules, seed):
    """The dual-tile kernel's top-1 pass without logits (32-column tree argmax, register-resident
    running max, padded columns at bo = -3e38) returns exactly the first maximum of the logits the
    same kernel writes on its general path: C spans one and several output passes, group ranges
    with a 16-column remainder and padding."""
    torch = require_cuda()
    R = ti.classbench_ruleset(fam, n_rules, seed)
    H = np.concatenate([ti.uniform_trace(R, 4000, seed + 1), ti.random_headers(131, seed + 2)])
    sigs, w, blob = model(R, N, 1, seed)
    ctx = T.Ctx(R, blob, mlp="bf16", kernel="dual")
    n = H.size
    out, pred = u32_dev(n), u32_dev(n)
    logits = torch.empty(n * len(sigs), dtype=torch.float32, device="cuda")
    fell = torch.zeros(n, dtype=torch.uint8, device="cuda")
    ctx.classify_ex(headers_dev(H), out, pred, logits, fell)
    out2, pred2 = u32_dev(n), u32_dev(n)
    ctx.classify_ex(headers_dev(H), out2, pred2, None, None)
    torch.cuda.synchronize()
    L = logits.cpu().numpy().reshape(n, -1)
    want = np.argmax(L, axis=1).astype(np.uint32)          # first maximum: ties -> lower index
    assert np.array_equal(u32_host(pred), want)
    assert np.array_equal(u32_host(pred2), want)
    assert np.array_equal(u32_host(out2), u32_host(out))
