// placement.cc — SLO-driven choice of the pipeline size (Algorithm 1) and contention-aware
// admission of simultaneous cold starts on shared host links (Eq. 3 / Eq. 4).  Host only.
//
// PAPER.md §4.1 Algorithm 1 (lines 420-452): enumerate s and w, predict TTFT / TPOT, keep the
// SLO-feasible choices, return the one with minimal GPU sharing, else (1, 1, (i_1)).
// PAPER.md §4.2 (lines 469-502): per server (here: per host-link group of GPUs, R17)
// record each cold-start worker's pending bytes S_i and deadline D_i; admit a new worker iff
// S_i <= B/(N+1) (D_i - T) for every worker including the new one (Eq. 3); on every membership
// change settle S_i' = S_i - B/N (T - T') and drop workers with S_i' < 0 (Eq. 4).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "../../include/hs.h"

namespace hs {
void set_error(const std::string& m);
}
using hs::set_error;

extern "C" hs_status hs_plan_auto(const hs_model_cfg* cfg, const hs_gpu* gpus, int32_t n_gpus,
                                  const hs_slo* slo, hs_plan* out, int32_t* sharing) {
  if (!cfg || !gpus || n_gpus <= 0 || !slo || !out) {
    set_error("hs_plan_auto: bad arguments");
    return HS_E_INVAL;
  }
  const int max_pp = std::max(1, std::min<int>(slo->max_pp > 0 ? slo->max_pp : 4, HS_MAX_STAGES));
  bool found = false;
  hs_plan best{};
  long best_share = 0;
  for (int s = 1; s <= std::min(max_pp, cfg->n_layers); ++s) {
    for (int w = 0; w <= s; ++w) {
      hs_plan p;
      if (hs_plan_stages(cfg, gpus, n_gpus, s, w, slo->t_prefill_s, slo->t_hop_s, &p) != HS_OK) continue;
      const double tpot = hs_predict_tpot_eq2(slo->t_decode_s, s, w, slo->t_hop_s);
      if (p.pred_ttft_s > slo->slo_ttft_s || tpot > slo->slo_tpot_s) continue;
      long share = 0;
      for (int k = 0; k < s; ++k)
        for (int i = 0; i < n_gpus; ++i)
          if (gpus[i].device == p.device[k]) share += gpus[i].n_workers;
      // minimal sharing; ties: smaller s, then larger w (cheaper consolidation, better TPOT)
      const bool better = !found || share < best_share ||
                          (share == best_share && (s < best.pp || (s == best.pp && w > [&] {
                                                     int bw = 0;
                                                     for (int k = 0; k < best.pp; ++k) bw += best.full_memory[k];
                                                     return bw;
                                                   }())));
      if (better) {
        found = true;
        best = p;
        best_share = share;
      }
    }
  }
  if (!found) {  // "Use single worker if no solution" (Algorithm 1)
    hs_status r = hs_plan_stages(cfg, gpus, n_gpus, 1, 1, slo->t_prefill_s, slo->t_hop_s, &best);
    if (r != HS_OK) return r;
    best_share = 0;
    for (int i = 0; i < n_gpus; ++i)
      if (gpus[i].device == best.device[0]) best_share = gpus[i].n_workers;
  }
  *out = best;
  if (sharing) *sharing = (int32_t)best_share;
  return found ? HS_OK : HS_E_INFEASIBLE;
}

struct LinkWorker {
  int64_t id;
  double pending, deadline;
};

struct hs_links {
  std::vector<double> bw;                    // B per group (bytes/s)
  std::vector<double> last;                  // T' per group
  std::vector<std::vector<LinkWorker>> ws;   // workers per group
  int64_t next_id = 1;
};

extern "C" hs_status hs_links_create(int32_t n_groups, const double* group_bytes_per_s, hs_links** out) {
  if (n_groups <= 0 || !group_bytes_per_s || !out) {
    set_error("hs_links_create: bad arguments");
    return HS_E_INVAL;
  }
  hs_links* l = new hs_links();
  l->bw.assign(group_bytes_per_s, group_bytes_per_s + n_groups);
  l->last.assign(n_groups, 0.0);
  l->ws.resize(n_groups);
  *out = l;
  return HS_OK;
}

static bool grp_ok(hs_links* l, int32_t g) { return l && g >= 0 && g < (int32_t)l->bw.size(); }

extern "C" hs_status hs_links_settle(hs_links* l, int32_t g, double now) {
  if (!grp_ok(l, g) || now < l->last[g]) {
    set_error("hs_links_settle: bad group or time going backwards");
    return HS_E_INVAL;
  }
  auto& v = l->ws[g];
  if (!v.empty()) {
    const double dec = l->bw[g] / (double)v.size() * (now - l->last[g]);  // Eq. 4
    for (auto& w : v) w.pending -= dec;
    v.erase(std::remove_if(v.begin(), v.end(), [](const LinkWorker& w) { return w.pending < 0.0; }), v.end());
  }
  l->last[g] = now;
  return HS_OK;
}

extern "C" hs_status hs_links_admit(hs_links* l, int32_t g, double pending, double deadline, double now,
                                    int32_t* accepted, int64_t* worker_id) {
  if (!grp_ok(l, g) || !accepted) {
    set_error("hs_links_admit: bad arguments");
    return HS_E_INVAL;
  }
  hs_status r = hs_links_settle(l, g, now);
  if (r != HS_OK) return r;
  auto& v = l->ws[g];
  const double share = l->bw[g] / (double)(v.size() + 1);
  bool ok = pending <= share * (deadline - now);  // Eq. 3 for the candidate
  for (const auto& w : v) ok = ok && w.pending <= share * (w.deadline - now);  // and every listed worker
  *accepted = ok ? 1 : 0;
  if (ok) {
    v.push_back({l->next_id, pending, deadline});
    if (worker_id) *worker_id = l->next_id;
    ++l->next_id;
  } else if (worker_id) {
    *worker_id = 0;
  }
  return HS_OK;
}

extern "C" hs_status hs_links_complete(hs_links* l, int32_t g, int64_t id, double now) {
  hs_status r = hs_links_settle(l, g, now);
  if (r != HS_OK) return r;
  auto& v = l->ws[g];
  v.erase(std::remove_if(v.begin(), v.end(), [&](const LinkWorker& w) { return w.id == id; }), v.end());
  return HS_OK;
}

extern "C" hs_status hs_links_pending(hs_links* l, int32_t g, int32_t max_n, int32_t* n, double* pending,
                                      int64_t* ids) {
  if (!grp_ok(l, g) || !n) {
    set_error("hs_links_pending: bad arguments");
    return HS_E_INVAL;
  }
  const auto& v = l->ws[g];
  *n = (int32_t)v.size();
  for (int i = 0; i < (int)v.size() && i < max_n; ++i) {
    if (pending) pending[i] = v[i].pending;
    if (ids) ids[i] = v[i].id;
  }
  return HS_OK;
}

extern "C" hs_status hs_links_destroy(hs_links* l) {
  delete l;
  return HS_OK;
}

// Contention-aware placement of one cold start (reading R20):
// Algorithm 1's selection on the contention-adjusted link view,
// Eq. 3 admission against the loads already streaming over each link group, Eq. 4
// bookkeeping.  For s = 1..max_pp the GPUs are ranked by 1/p'_i with
// p'_i = min(p_i, B_g / (N_g + 1)) (the bandwidth a new load on GPU i would get; ties -> fewer
// loads N_g on its group), all stages low-memory (w = 0: a burst of cold starts, no
// consolidation).  Each stage k on group g gets the equal credit p_eff = min(p_k, B_g / (N_g + s_g))
// (s_g: the candidate's stages on g), so TTFT_pred(s) = max_k bytes_k / p_eff_k (Eq. 5 as in R9,
// with the fetching term replaced by the contended link).  A candidate is admissible iff every
// worker already on a touched group still meets its deadline under the new share (Eq. 3 with
// N + s_g) and TTFT_pred <= SLO.  The admissible candidate with the smallest prediction wins
// (ties: smaller s); if none, the smallest prediction.  Its stages are then recorded as workers
// (pending = stage bytes, deadline D = T + TTFT_pred, "the fetching deadline comes from the
// prediction of TTFT").
extern "C" hs_status hs_place_cold_start(const hs_model_cfg* cfg, const hs_gpu* gpus, int32_t n_gpus, hs_links* l,
                                         double now, double slo_ttft_s, int32_t max_pp, hs_plan* out,
                                         double* pred_ttft_s, int32_t* admitted, int64_t* worker_ids) {
  if (!cfg || !gpus || n_gpus <= 0 || !l || !out) {
    set_error("hs_place_cold_start: bad arguments");
    return HS_E_INVAL;
  }
  std::vector<int> seen;
  for (int i = 0; i < n_gpus; ++i) {
    const int g = gpus[i].link_group;
    if (!grp_ok(l, g) || gpus[i].h2d_gbps <= 0) {
      set_error("hs_place_cold_start: a GPU's link group is not in the registry");
      return HS_E_INVAL;
    }
    if (std::find(seen.begin(), seen.end(), g) == seen.end()) {
      seen.push_back(g);
      hs_status r = hs_links_settle(l, g, now);  // Eq. 4 up to T
      if (r != HS_OK) return r;
    }
  }
  auto N = [&](int g) { return (double)l->ws[g].size(); };
  std::vector<hs_gpu> view(gpus, gpus + n_gpus);
  for (auto& v : view) {
    v.h2d_gbps = std::min(v.h2d_gbps, l->bw[v.link_group] / 1e9 / (N(v.link_group) + 1.0));
    v.n_workers = (int32_t)N(v.link_group);
  }
  auto gpu_of = [&](int dev) {
    for (int i = 0; i < n_gpus; ++i)
      if (gpus[i].device == dev) return i;
    return -1;
  };
  bool have = false, best_ok = false;
  double best_pred = 0;
  hs_plan best{};
  const int smax = std::max(1, std::min<int>({max_pp > 0 ? max_pp : 4, HS_MAX_STAGES, cfg->n_layers, n_gpus}));
  for (int s = 1; s <= smax; ++s) {
    hs_plan p;
    if (hs_plan_stages(cfg, view.data(), n_gpus, s, 0, 0.0, 0.0, &p) != HS_OK) continue;
    std::map<int, int> sg;  // stages per group
    for (int k = 0; k < s; ++k) sg[gpus[gpu_of(p.device[k])].link_group]++;
    double pred = 0;
    for (int k = 0; k < s; ++k) {
      const hs_gpu& gk = gpus[gpu_of(p.device[k])];
      const int g = gk.link_group;
      const double peff = std::min(gk.h2d_gbps * 1e9, l->bw[g] / (N(g) + sg[g]));
      pred = std::max(pred, (double)p.stage_bytes[k] / peff);
    }
    bool ok = pred <= slo_ttft_s;
    for (auto& kv : sg) {  // Eq. 3 for every worker already on the group, under the new share
      const double share = l->bw[kv.first] / (N(kv.first) + kv.second);
      for (const auto& w : l->ws[kv.first]) ok = ok && w.pending <= share * (w.deadline - now);
    }
    const bool better = !have || (ok && !best_ok) || (ok == best_ok && pred < best_pred);
    if (better) {
      have = true;
      best_ok = ok;
      best_pred = pred;
      best = p;
    }
  }
  if (!have) {
    set_error("hs_place_cold_start: no GPU set can hold the model");
    return HS_E_INFEASIBLE;
  }
  best.pred_ttft_s = best_pred;
  for (int k = 0; k < best.pp; ++k) {  // record the stages as cold-start workers of their groups
    const int g = gpus[gpu_of(best.device[k])].link_group;
    l->ws[g].push_back({l->next_id, (double)best.stage_bytes[k], now + best_pred});
    if (worker_ids) worker_ids[k] = l->next_id;
    ++l->next_id;
  }
  *out = best;
  if (pred_ttft_s) *pred_ttft_s = best_pred;
  if (admitted) *admitted = best_ok ? 1 : 0;
  return HS_OK;
}
