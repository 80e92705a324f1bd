"""Plain PyTorch trainer of TaNG's tuple predictor -- setup, off the hot path.

P:389-394 (§6.2): training records D = <s_1..s_k, tuple_idx>, the label being the tuple of
the highest-priority matching rule of a historical packet; classes with fewer than alpha
samples are oversampled up to alpha; cross-entropy + Adam, batch 8192, LR 1e-3 decayed x0.1
every 200 epochs (scaled here to a wall-clock budget: the decay points are placed at the same
fractions of the run), and alpha x10 with a retrain when the accuracy stays below beta.

Labels come from libtang itself: tang_classify_with_pred with k = 0 searches every tuple,
i.e. returns the brute-force winner on the GPU.  Every rule of a
fresh build sits in its exact-signature tuple, so the label is that rule's signature index.
The network is trained with the inference quantisation points (bf16 GEMM inputs under
autocast, fp32 layer 0), then exported as fp32 [in][out] weights for the model blob.
"""
from __future__ import annotations

import math
import time

import numpy as np
import torch

from . import tang as T


def tuple_signatures(rules: np.ndarray):
    """Class order of a fresh model (SURVEY.md §8(c) reading 8): the distinct
    (sip_len, dip_len) signatures in order of first occurrence in the rule file.  The trainer
    writes this list into the blob; libtang takes the tuple set from the blob, never from here."""
    code = rules["sip_len"].astype(np.int64) * 64 + rules["dip_len"].astype(np.int64)
    uniq, first = np.unique(code, return_index=True)
    return [(int(c // 64), int(c % 64)) for c in uniq[np.argsort(first)]]


class TangMLP(torch.nn.Module):
    """Input FC + ReLU, B residual blocks B(x) = A(A(x.w1+b1).w2 + b2 + x), output FC (Eq. 1)."""

    def __init__(self, S, N, B, C):
        super().__init__()
        self.l0 = torch.nn.Linear(S, N)
        self.l1 = torch.nn.ModuleList(torch.nn.Linear(N, N) for _ in range(B))
        self.l2 = torch.nn.ModuleList(torch.nn.Linear(N, N) for _ in range(B))
        self.lo = torch.nn.Linear(N, C)
        with torch.no_grad():
            self.l0.weight.mul_(8.0)            # inputs are 16-bit chunks / 65536 in [0, 1)
            for l in self.l2:
                l.weight.mul_(0.5)

    def forward(self, x, act_exp=None):
        if act_exp is not None:
            return self.forward_nvfp4(x, act_exp)
        h = torch.relu(self.l0(x.float()))
        with torch.autocast("cuda", dtype=torch.bfloat16, enabled=x.is_cuda):
            for a, b in zip(self.l1, self.l2):
                h = torch.relu(b(torch.relu(a(h))) + h)
            return self.lo(h).float()

    def forward_nvfp4(self, x, act_exp):
        """Quantisation-aware forward of the NVFP4 chain (R24, fake quantisation with a
        straight-through gradient): W1, W2, Wo and the GEMM inputs h0, u_b, h_b are quantised to e2m1
        codes with e4m3 scales per 16 along K under their power-of-two tensor scales (activations:
        the calibrated exponents act_exp); layer 0 stays fp32 (R22); bias, skip and ReLU in fp32."""
        ste = lambda v, q: v + (q - v).detach()
        qw = lambda W: ste(W, nvfp4_fake(W, pow2_exp(float(W.detach().abs().max()))))
        qa = lambda v, e: ste(v, nvfp4_fake(v, e))
        h = torch.relu(self.l0(x.float()))
        hq = qa(h, act_exp[0])
        for i, (a, b) in enumerate(zip(self.l1, self.l2)):
            u = torch.relu(torch.nn.functional.linear(hq, qw(a.weight), a.bias))
            uq = qa(u, act_exp[1 + 2 * i])
            h = torch.relu(torch.nn.functional.linear(uq, qw(b.weight), b.bias) + hq)
            hq = qa(h, act_exp[2 + 2 * i])
        return torch.nn.functional.linear(hq, qw(self.lo.weight), self.lo.bias)

    @torch.no_grad()
    def load(self, w: dict):
        """Warm start from exported fp32 weights ([in][out]) -- incremental training."""
        t = lambda a: torch.as_tensor(a, dtype=torch.float32, device=self.l0.weight.device)
        self.l0.weight.copy_(t(w["W0"]).T)
        self.l0.bias.copy_(t(w["b0"]))
        for i in range(len(self.l1)):
            self.l1[i].weight.copy_(t(w["W1"][i]).T)
            self.l1[i].bias.copy_(t(w["b1"][i]))
            self.l2[i].weight.copy_(t(w["W2"][i]).T)
            self.l2[i].bias.copy_(t(w["b2"][i]))
        self.lo.weight.copy_(t(w["Wo"]).T)
        self.lo.bias.copy_(t(w["bo"]))

    def export(self) -> dict:
        g = lambda t: t.detach().float().cpu().numpy()
        return dict(S=self.l0.in_features, N=self.l0.out_features, B=len(self.l1), C=self.lo.out_features,
                    W0=g(self.l0.weight).T.copy(), b0=g(self.l0.bias),
                    W1=[g(l.weight).T.copy() for l in self.l1], b1=[g(l.bias) for l in self.l1],
                    W2=[g(l.weight).T.copy() for l in self.l2], b2=[g(l.bias) for l in self.l2],
                    Wo=g(self.lo.weight).T.copy(), bo=g(self.lo.bias))


def features_torch(hdr_u8: torch.Tensor) -> torch.Tensor:
    """The 7 segments / 65536 of headers given as a uint8 [n*16] device tensor."""
    w = hdr_u8.view(torch.int32).view(-1, 4).long() & 0xFFFFFFFF
    sip, dip, ports, proto = w[:, 0], w[:, 1], w[:, 2], w[:, 3] & 0xFF
    seg = torch.stack([sip >> 16, sip & 0xFFFF, dip >> 16, dip & 0xFFFF, ports & 0xFFFF, ports >> 16, proto], 1)
    return seg.float() / 65536.0


def rule_tuple_map(rules: np.ndarray, sigs) -> tuple[np.ndarray, np.ndarray]:
    """(sorted rule ids, tuple index of each) for rules placed at their exact signature."""
    idx = {s: j for j, s in enumerate(sigs)}
    tup = np.array([idx[(int(a), int(b))] for a, b in zip(rules["sip_len"], rules["dip_len"])], dtype=np.int64)
    order = np.argsort(rules["id"])
    return rules["id"][order].astype(np.int64), tup[order]


def gpu_labels(ctx: T.Ctx, hdr_u8: torch.Tensor, rules, sigs, chunk=1 << 20, placed=False) -> torch.Tensor:
    """Tuple of the brute-force winner (k = 0 search on the GPU); -1 for unmatched packets.
    placed=True asks the ctx where each rule lives (after restricted inserts, a rule can
    sit in a tuple other than its own signature's)."""
    n = hdr_u8.numel() // 16
    out = torch.empty(n, dtype=torch.int32, device=hdr_u8.device)
    for o in range(0, n, chunk):
        m = min(chunk, n - o)
        ctx.classify_with_pred(hdr_u8[o * 16:(o + m) * 16], None, 0, out[o:o + m])
    if placed:
        order = np.argsort(rules["id"])
        ids = rules["id"][order].astype(np.int64)
        tup = np.array([ctx.rule_tuple(int(i)) for i in ids], dtype=np.int64)
    else:
        ids, tup = rule_tuple_map(rules, sigs)
    ids_t = torch.from_numpy(ids).to(hdr_u8.device)
    tup_t = torch.from_numpy(tup).to(hdr_u8.device)
    rid = out.long() & 0xFFFFFFFF
    pos = torch.searchsorted(ids_t, rid).clamp(max=ids_t.numel() - 1)
    return torch.where(ids_t[pos] == rid, tup_t[pos], torch.full_like(rid, -1))


def torch_labels(rules: np.ndarray, sigs, hdr_u8: torch.Tensor, chunk: int = 256) -> torch.Tensor:
    """Training labels without libtang (the label of a historical packet is the tuple of
    its highest-priority matching rule): a plain brute-force scan in torch on the headers' device,
    rules sorted by (priority, id) so the first matching column wins; -1 for unmatched packets.
    Used for the committed models (scripts/train_model.py), whose weights are also oracle inputs,
    so no input of the oracle passes through the CUDA library.  Rules sit at their exact signature."""
    dev = hdr_u8.device
    order = np.lexsort((rules["id"], rules["priority"]))
    R = rules[order]
    idx = {s: j for j, s in enumerate(sigs)}
    tup = torch.tensor([idx[(int(a), int(b))] for a, b in zip(R["sip_len"], R["dip_len"])], device=dev)
    i32 = lambda a: torch.from_numpy(np.ascontiguousarray(a).astype(np.int64)).to(dev)

    def mask(l):
        l = i32(l)
        return torch.where(l == 0, torch.zeros_like(l), (0xFFFFFFFF << (32 - l)) & 0xFFFFFFFF)
    ms, md = mask(R["sip_len"]), mask(R["dip_len"])
    rs, rd = i32(R["sip"]) & ms, i32(R["dip"]) & md
    spl, sph, dpl, dph = i32(R["sp_lo"]), i32(R["sp_hi"]), i32(R["dp_lo"]), i32(R["dp_hi"])
    pm = i32(R["proto_mask"])
    pv = i32(R["proto"]) & pm
    w = hdr_u8.view(torch.int32).view(-1, 4).long() & 0xFFFFFFFF
    n = w.shape[0]
    out = torch.empty(n, dtype=torch.long, device=dev)
    for o in range(0, n, chunk):
        h = w[o:o + chunk]
        s, d = h[:, 0:1], h[:, 1:2]
        sp, dp, pr = h[:, 2:3] & 0xFFFF, h[:, 2:3] >> 16, h[:, 3:4] & 0xFF
        m = ((s & ms) == rs) & ((d & md) == rd) & (sp >= spl) & (sp <= sph) & (dp >= dpl) & (dp <= dph) \
            & ((pr & pm) == pv)
        first = m.to(torch.uint8).argmax(1)                 # first maximum = first matching rule
        out[o:o + chunk] = torch.where(m.any(1), tup[first], torch.full_like(first, -1))
    return out


def oversample(labels: torch.Tensor, alpha: int, gen: torch.Generator) -> torch.Tensor:
    """Indices of the training set after raising every present class below alpha to alpha
    samples by repetition; absent classes stay absent."""
    valid = torch.nonzero(labels >= 0).squeeze(1)
    lab = labels[valid]
    counts = torch.bincount(lab)
    parts = [valid]
    for c in torch.nonzero((counts > 0) & (counts < alpha)).squeeze(1).tolist():
        members = valid[lab == c]
        need = alpha - members.numel()
        parts.append(members[torch.arange(need, device=labels.device) % members.numel()])
    return torch.cat(parts)


def train(rules, sigs, N, B, hdr_u8: torch.Tensor, labels: torch.Tensor, seconds=60.0, alpha=1000,
          beta=0.95, batch=8192, lr=1e-3, seed=0, log=None, init: dict | None = None,
          max_rounds: int = 2, act_exp: list | None = None) -> tuple[dict, float]:
    """Train until the wall-clock budget ends; returns (fp32 weights, training accuracy).
    `init` warm-starts from existing weights (incremental training of the deferred update)."""
    dev = hdr_u8.device
    torch.manual_seed(seed)
    gen = torch.Generator(device=dev)
    gen.manual_seed(seed)
    X = features_torch(hdr_u8)
    model = TangMLP(7, N, B, len(sigs)).to(dev)
    if init is not None:
        model.load(init)
    acc = 0.0
    t0 = time.time()
    rounds = 0
    while rounds < max_rounds:
        idx = oversample(labels, alpha, gen)
        opt = torch.optim.Adam(model.parameters(), lr=lr)
        # the wall-clock budget is shared by max_rounds rounds (each with the LR schedule); after a
        # round whose accuracy stays below beta, alpha is raised x10 before the next.  A
        # round that starts late (the previous one overran) still runs at least one chunk of steps.
        budget = max((seconds - (time.time() - t0)) / (max_rounds - rounds), 1e-3)
        t_round = time.time()
        step = 0
        while step == 0 or time.time() - t_round < budget:
            frac = (time.time() - t_round) / budget
            for g in opt.param_groups:                      # x0.1 at 20/40/60/80% (200/1000 epochs)
                g["lr"] = lr * (0.1 ** int(frac * 5))
            perm = idx[torch.randint(0, idx.numel(), (batch * 16,), device=dev, generator=gen)]
            for b in range(16):
                sel = perm[b * batch:(b + 1) * batch]
                loss = torch.nn.functional.cross_entropy(model(X[sel], act_exp), labels[sel])
                opt.zero_grad(set_to_none=True)
                loss.backward()
                opt.step()
                step += 1
        rounds += 1
        acc = evaluate(model, X, labels, act_exp=act_exp)
        if log:
            log(f"train round {rounds}: alpha={alpha} steps={step} acc={acc:.4f} t={time.time() - t0:.1f}s")
        if acc < beta:
            alpha *= 10                                      # below beta, retrain with alpha x10
    return model.export(), acc


@torch.no_grad()
def evaluate(model, X, labels, chunk=1 << 18, act_exp=None) -> float:
    ok = tot = 0
    for o in range(0, X.shape[0], chunk):
        lab = labels[o:o + chunk]
        m = lab >= 0
        p = model(X[o:o + chunk], act_exp).argmax(1)
        ok += int((p[m] == lab[m]).sum())
        tot += int(m.sum())
    return ok / max(1, tot)


_E2M1_GRID = (0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0)
_E2M1_MIDS = (0.25, 0.75, 1.25, 1.75, 2.5, 3.5, 5.0)


def nvfp4_fake(v: torch.Tensor, e: int) -> torch.Tensor:
    """NVFP4 fake quantisation along the last axis (R24): v / 2^e in blocks of 16, block scale
    sf = e4m3(max|.| / 6), codes = nearest e2m1 value of v / (2^e sf) (saturating; ties go to the
    smaller magnitude -- the trainer only needs the rounding grid, the kernel and the oracle round
    to nearest even), dequantised back.  The last axis must be a multiple of 16."""
    shp = v.shape
    s = math.ldexp(1.0, e)
    b = (v / s).reshape(*shp[:-1], shp[-1] // 16, 16)
    # (clamped to e4m3's 448: during fine-tuning activations may outgrow their calibrated scale)
    sf = (b.abs().amax(dim=-1, keepdim=True) / 6.0).clamp(max=448.0).to(torch.float8_e4m3fn).float()
    safe = torch.where(sf > 0, sf, torch.ones_like(sf))
    a = (b.abs() / safe).clamp(max=6.0)
    grid = torch.tensor(_E2M1_GRID, device=v.device, dtype=torch.float32)
    mids = torch.tensor(_E2M1_MIDS, device=v.device, dtype=torch.float32)
    q = torch.sign(b) * grid[torch.bucketize(a.contiguous(), mids)] * sf
    return (q * s).reshape(shp)


def pow2_exp(amax: float) -> int:
    return _pow2_exp(amax)


def _pow2_exp(amax: float) -> int:
    """Smallest e with amax <= 448 * 2^e (e4m3 max 448), exact comparisons (R23)."""
    if not amax > 0:
        return 0
    e = math.frexp(amax)[1] - 9
    for _ in range(3):
        if amax > math.ldexp(448.0, e):
            e += 1
        if amax <= math.ldexp(448.0, e - 1):
            e -= 1
    return e


@torch.no_grad()
def calibrate_fp8(w: dict, X: torch.Tensor, chunk: int = 1 << 18) -> list:
    """Static per-layer activation scales for the fp8 chain (TensorRT-style max calibration,
    P:304 "precision quantization"; R23): the fp32 network is run on a calibration
    sample X [n, 7] and each of h0, u_1, h_1, ..., u_B, h_B gets the power-of-two scale whose
    e4m3 range (448 * 2^e) covers its maximum.  Returns the 2B+1 exponents for pack_blob."""
    dev = X.device
    t = lambda a: torch.as_tensor(np.asarray(a), dtype=torch.float32, device=dev)
    B = int(w["B"])
    amax = [0.0] * (2 * B + 1)
    for o in range(0, X.shape[0], chunk):
        x = X[o:o + chunk].float()
        h = torch.relu(x @ t(w["W0"]) + t(w["b0"]))
        amax[0] = max(amax[0], float(h.max()))
        for i in range(B):
            u = torch.relu(h @ t(w["W1"][i]) + t(w["b1"][i]))
            h = torch.relu(u @ t(w["W2"][i]) + t(w["b2"][i]) + h)
            amax[1 + 2 * i] = max(amax[1 + 2 * i], float(u.max()))
            amax[2 + 2 * i] = max(amax[2 + 2 * i], float(h.max()))
    return [_pow2_exp(a) for a in amax]



def round_weights_bf16(w: dict) -> dict:
    """W1, W2, Wo rounded to bf16 (RNE, torch's cast) -- the form a committed model is stored in
    (tang_inputs.save_model); the bf16 chain rounds them there anyway (R5)."""
    bf = lambda a: torch.as_tensor(np.asarray(a, np.float32)).to(torch.bfloat16).float().numpy()
    out = dict(w)
    out["W1"] = [bf(x) for x in w["W1"]]
    out["W2"] = [bf(x) for x in w["W2"]]
    out["Wo"] = bf(w["Wo"])
    return out
