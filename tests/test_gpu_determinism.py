"""Race detection by repetition (compute-sanitizer is closed on this pool since round 2,
profiles/r02g_sanitize_closed.txt).  Every tcgen05 chain fixes its accumulation order, so a correct
kernel returns bit-identical logits, predictions and rule ids on every launch; a race between the TMA
ring, the MMA issuer, the epilogue warps, the 2SM peer's forwarder warp or the cross-CTA barriers
shows up as a launch whose bits differ.  Each variant runs many launches over a batch that spans every
CTA of the persistent grid several times, plus a ragged tail."""
import numpy as np
import pytest

import tang_inputs as ti
from oracle import tss as otss
from tests._helpers import headers_dev, require_cuda

pytestmark = pytest.mark.gpu

CASES = [  # (mlp, kernel, N, B)
    ("bf16", "2sm", 512, 6),
    ("bf16", "2sm", 256, 2),
    ("bf16", "single", 512, 2),
    ("bf16", "wide", 256, 2),
    ("bf16", "dual", 256, 2),
    ("bf16", "dual", 128, 4),
    ("fp8", "auto", 512, 2),
    ("fp8", "auto", 256, 2),
    ("nvfp4", "auto", 256, 2),
]


@pytest.mark.parametrize("mlp,kernel,N,B", CASES)
def test_repeated_launches_are_bit_identical(mlp, kernel, N, B):
    torch = require_cuda()
    from paper_2601_03187_b200 import tang as T, train as TR
    R = ti.classbench_ruleset("acl", 4000, 17)
    n = 148 * 128 * 3 + 77                          # three tiles per CTA of the full grid + a ragged tail
    H = np.concatenate([ti.uniform_trace(R, n - 500, 18), ti.random_headers(500, 19)])
    sigs = otss.signatures_first_occurrence(R)
    w = ti.random_weights(7, N, B, len(sigs), seed=N + B)
    if mlp in ("fp8", "nvfp4"):
        w["act_exp"] = TR.calibrate_fp8(w, TR.features_torch(torch.from_numpy(H.view(np.uint8).copy())))
    ctx = T.Ctx(R, T.pack_blob(sigs, w), mlp=mlp, kernel=kernel)
    d = headers_dev(H)
    C = len(sigs)
    ref_out = ref_pred = ref_lg = None
    bad = 0
    for it in range(40):
        out = torch.empty(n, dtype=torch.int32, device="cuda")
        pred = torch.empty(n, dtype=torch.int32, device="cuda")
        lg = torch.empty(n * C, dtype=torch.float32, device="cuda")
        if it % 2:
            ctx.classify_ex(d, out, pred, lg)      # logits written (top-k + logits epilogue)
        else:
            ctx.classify_ex(d, out, pred)          # fast top-1 epilogue
        torch.cuda.synchronize()
        o, p = out.cpu().numpy(), pred.cpu().numpy()
        if ref_out is None:
            ref_out, ref_pred = o, p
        else:
            bad += int((o != ref_out).sum() + (p != ref_pred).sum())
        if it % 2:
            l = lg.cpu().numpy().view(np.uint32)
            if ref_lg is None:
                ref_lg = l
            else:
                bad += int((l != ref_lg).sum())
    ctx.close()
    assert bad == 0, f"{mlp}/{kernel} N={N} B={B}: {bad} values differ between launches"
