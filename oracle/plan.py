"""Oracle stage planning: layer split, stage bytes, the paper's predictors and server choice.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

  * Eq. 1: TTFT = t_c + (M/s) max_i(1/b_i + 1/p_i) + t_p (s - w + w/s) + t_n s
  * Eq. 2: TPOT = t_d (s - w + w/s) + t_n s
  * Eq. 5: TTFT = max_i( t_cc + t_cu + max((M/s)/p_i, t_l), (M/s)/b_i )
                                      + t_p (s - w + w/s) + t_n s
  * selection: the w full-memory workers take the servers with the
    smallest 1/b + 1/p among those that fit the whole model; the rest are merged with the
    low-memory-capable servers and the smallest s - w ratios are taken.
  * DESIGN.md reading R9: on one box there is no remote fetch (1/b = 0), runtime/library
    terms are paid before T0 (t_cc = t_cu = t_l = 0), and each stage's own byte count
    replaces M/s, so  TTFT_pred = max_k(bytes_k / p_k) + t_p (s - w + w/s) + t_n s.
"""
from __future__ import annotations

from .decoder import embed_param_bytes, final_param_bytes, layer_param_bytes, split_layers


def eq1_ttft(t_c, M, s, w, b, p, t_p, t_n):
    return t_c + (M / s) * max(1.0 / bi + 1.0 / pi for bi, pi in zip(b, p)) + t_p * (s - w + w / s) + t_n * s


def eq2_tpot(t_d, s, w, t_n):
    return t_d * (s - w + w / s) + t_n * s


def eq5_ttft(t_cc, t_cu, t_l, M, s, w, b, p, t_p, t_n):
    fetch = max(max(t_cc + t_cu + max((M / s) / pi, t_l), (M / s) / bi) for bi, pi in zip(b, p))
    return fetch + t_p * (s - w + w / s) + t_n * s


def select_servers(full_capable, low_capable, s, w):
    """full_capable / low_capable: lists of (server_id, ratio[, n_workers]).  Returns s server
    ids: the w smallest-ratio full-capable, then the s-w smallest-ratio of the merged rest;
    ratio ties broken by fewer running workers (R18), then server id."""
    key = lambda t: (t[1], t[2] if len(t) > 2 else 0, t[0])  # noqa: E731
    fc = sorted(full_capable, key=key)
    if len(fc) < w:
        raise ValueError("infeasible")
    first = fc[:w]
    rest = sorted(list(low_capable) + fc[w:], key=key)
    if len(rest) < s - w:
        raise ValueError("infeasible")
    return [t[0] for t in first + rest[: s - w]]


def stage_param_bytes(cfg: dict, pp: int):
    """Bytes each stage must load (no padding): its layers, + embedding on stage 0,
    + final norm and lm_head on the last stage."""
    out = []
    for k, (b, e) in enumerate(split_layers(cfg["n_layers"], pp)):
        n = (e - b) * layer_param_bytes(cfg)
        if k == 0:
            n += embed_param_bytes(cfg)
        if k == pp - 1:
            n += final_param_bytes(cfg)
        out.append(n)
    return out


def plan(cfg: dict, gpus, pp: int, full_memory_stages: int = 1, t_prefill_s=0.0, t_hop_s=0.0):
    """gpus: list of dicts {device, h2d_gbps, link_group, free_bytes}.  Mirrors hs_plan_stages:
    w = full_memory_stages stages reserve the whole model (stage 0 first), chosen by the
    selection rule with ratio 1/p; returns dict(pp, device, ranges, stage_bytes,
    full_memory, pred_ttft_s)."""
    if pp > cfg["n_layers"]:
        raise ValueError("infeasible")
    sb = stage_param_bytes(cfg, pp)
    model_bytes = embed_param_bytes(cfg) + final_param_bytes(cfg) + cfg["n_layers"] * layer_param_bytes(cfg)
    w = min(full_memory_stages, pp)
    full = [(g["device"], 1.0 / g["h2d_gbps"], g.get("n_workers", 0)) for g in gpus if g["free_bytes"] >= model_bytes]
    low = [(g["device"], 1.0 / g["h2d_gbps"], g.get("n_workers", 0)) for g in gpus
           if max(sb) <= g["free_bytes"] < model_bytes]
    devs = select_servers(full, low, pp, w)
    p = {g["device"]: g["h2d_gbps"] for g in gpus}
    pred = max(sb[k] / (p[devs[k]] * 1e9) for k in range(pp)) + t_prefill_s * (pp - w + w / pp) + t_hop_s * pp
    return dict(pp=pp, device=devs, ranges=split_layers(cfg["n_layers"], pp), stage_bytes=sb,
                full_memory=[1 if k < w else 0 for k in range(pp)], pred_ttft_s=pred)


def alg1(cfg: dict, gpus, t_p, t_d, t_n, slo_ttft, slo_tpot, max_pp=4):
    """Algorithm 1 by exhaustive enumeration on one box: every (s, w) whose
    selected GPUs exist and whose predicted TTFT (Eq. 5 specialised, R9) and TPOT (Eq. 2) meet
    the SLOs is feasible; return the feasible choice with minimal GPU sharing (workers already
    on the chosen GPUs), ties -> smaller s, then larger w; else the single-worker fallback.
    Returns (plan, sharing, feasible)."""
    best = None
    for s in range(1, min(max_pp, cfg["n_layers"]) + 1):
        for w in range(0, s + 1):
            try:
                p = plan(cfg, gpus, s, w, t_p, t_n)
            except ValueError:
                continue
            if p["pred_ttft_s"] > slo_ttft or eq2_tpot(t_d, s, w, t_n) > slo_tpot:
                continue
            nw = {g["device"]: g.get("n_workers", 0) for g in gpus}
            share = sum(nw[d] for d in p["device"])
            key = (share, s, -w)
            if best is None or key < best[0]:
                best = (key, p, share)
    if best is None:
        p = plan(cfg, gpus, 1, 1, t_p, t_n)
        nw = {g["device"]: g.get("n_workers", 0) for g in gpus}
        return p, nw[p["device"][0]], False
    return best[1], best[2], True


class ContentionRegistry:
    """Eq. 3 / Eq. 4 for one server (here: one host-link group), exactly as
    written: admit iff S_i <= B/(N+1) (D_i - T) for all workers incl. the candidate; on each
    change S_i' = S_i - B/N (T - T'), deleting workers with S_i' < 0."""

    def __init__(self, B):
        self.B, self.last, self.ws, self.next = B, 0.0, {}, 1

    def settle(self, now):
        assert now >= self.last
        if self.ws:
            dec = self.B / len(self.ws) * (now - self.last)
            self.ws = {i: (S - dec, D) for i, (S, D) in self.ws.items() if S - dec >= 0}
        self.last = now

    def admit(self, S, D, now):
        self.settle(now)
        share = self.B / (len(self.ws) + 1)
        ok = S <= share * (D - now) and all(Si <= share * (Di - now) for Si, Di in self.ws.values())
        if not ok:
            return False, 0
        wid = self.next
        self.next += 1
        self.ws[wid] = (S, D)
        return True, wid

    def complete(self, wid, now):
        self.settle(now)
        self.ws.pop(wid, None)

    def record(self, S, D):
        """A placed cold-start worker enters the list (pending S, deadline D)."""
        wid = self.next
        self.next += 1
        self.ws[wid] = (S, D)
        return wid


def place_cold_start(cfg: dict, gpus, regs: dict, now: float, slo_ttft: float, max_pp: int = 4):
    """Contention-aware placement of one cold start (reading R20), written out from
    Algorithm 1, Eq. 3 and Eq. 4:
      1. settle every link group to `now` (Eq. 4);
      2. for s = 1..max_pp: Alg. 1's GPU selection with w = 0 on the contended links
         p'_i = min(p_i, B_g / (N_g + 1)) (ties: fewer loads N_g, then device id);
      3. stage k on group g gets p_eff = min(p_k, B_g / (N_g + s_g)); TTFT_pred = max_k bytes_k / p_eff;
      4. admissible iff TTFT_pred <= SLO and Eq. 3 holds for every worker on a touched group with
         N + s_g workers;
      5. the admissible choice with the smallest TTFT_pred (ties: smaller s), else the smallest;
      6. its stages are recorded (pending = stage bytes, deadline = now + TTFT_pred).
    gpus: dicts {device, h2d_gbps, link_group, free_bytes}; regs: group -> ContentionRegistry
    (B in bytes/s).  Returns (plan dict, pred, admitted, worker ids)."""
    for g in sorted({x["link_group"] for x in gpus}):
        regs[g].settle(now)
    N = {g: len(r.ws) for g, r in regs.items()}
    view = [dict(x, h2d_gbps=min(x["h2d_gbps"], regs[x["link_group"]].B / 1e9 / (N[x["link_group"]] + 1)),
                 n_workers=N[x["link_group"]]) for x in gpus]
    by_dev = {x["device"]: x for x in gpus}
    best = None
    for s in range(1, min(max_pp, cfg["n_layers"], len(gpus)) + 1):
        try:
            p = plan(cfg, view, s, 0)
        except ValueError:
            continue
        sg = {}
        for d in p["device"]:
            g = by_dev[d]["link_group"]
            sg[g] = sg.get(g, 0) + 1
        pred = max(p["stage_bytes"][k] / min(by_dev[d]["h2d_gbps"] * 1e9,
                                             regs[by_dev[d]["link_group"]].B / (N[by_dev[d]["link_group"]] + sg[by_dev[d]["link_group"]]))
                   for k, d in enumerate(p["device"]))
        ok = pred <= slo_ttft
        for g, n in sg.items():
            share = regs[g].B / (N[g] + n)
            ok = ok and all(S <= share * (D - now) for S, D in regs[g].ws.values())
        key = (0 if ok else 1, pred, s)
        if best is None or key < best[0]:
            best = (key, p, pred, ok)
    if best is None:
        raise ValueError("infeasible")
    _, p, pred, ok = best
    ids = [regs[by_dev[d]["link_group"]].record(p["stage_bytes"][k], now + pred) for k, d in enumerate(p["device"])]
    return p, pred, ok, ids
