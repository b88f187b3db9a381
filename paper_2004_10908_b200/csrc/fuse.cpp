// fuse.cpp -- create-time planning of multi-layer passes ("model
// decomposition": the paper's LSDNN kernel is "model decomposition-based",
// PAPER.md:2560-2562; here the decomposition is by connected components of
// consecutive layers so that one HBM pass can run several layers on chip).
//
// Nodes are (boundary b, neuron) for b = 0..m (boundary b = input of layer
// a+b).  Every group of layer a+b joins its sources (boundary b) and its member
// columns (boundary b+1).  A pass [a, a+m) is feasible when every connected
// component has at most `cap` nodes on every boundary; the greedy planner
// extends a pass layer by layer while that holds.
#include <algorithm>
#include <array>
#include <cmath>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <thread>

#include "sdnn_internal.h"

namespace sdnn {
namespace {

struct UF {
  std::vector<int32_t> parent;
  void init(int64_t nodes) {
    parent.resize(nodes);
    std::iota(parent.begin(), parent.end(), 0);
  }
  int32_t find(int32_t x) {
    while (parent[x] != x) {
      parent[x] = parent[parent[x]];
      x = parent[x];
    }
    return x;
  }
  void unite(int32_t x, int32_t y) {
    x = find(x);
    y = find(y);
    if (x == y) return;
    if (x > y) std::swap(x, y);
    parent[y] = x;
  }
};

// general: per-slot (non-uniform) layers may be fused too (blocked plans only:
// k_pass_gw is their only pass kernel); a lane reads 8 members' weights of a
// term as two float4 of a 32-member row, hence gmax == 32
bool fusable(const PackedLayer &p, bool general = false) {
  return (p.uniform || (general && p.gmax == 32)) && p.kmax <= 32 && p.gmax <= 32;
}

// a layer whose groups can overwrite their own source slots: every source row
// feeds at most one group, and no group has more members than sources
bool inplace(const PackedLayer &p) {
  std::vector<uint8_t> seen(p.n, 0);
  for (int32_t g = 0; g < p.ngroups; ++g) {
    if (p.gg[g] > p.gk[g]) return false;
    for (int t = 0; t < p.gk[g]; ++t) {
      uint8_t &s = seen[p.src[(size_t)g * p.kmax + t]];
      if (s) return false;
      s = 1;
    }
  }
  return true;
}

// join layer (boundary b -> b+1) into the union-find
void add_layer(UF &uf, const PackedLayer &p, int32_t n, int b) {
  const int64_t in0 = (int64_t)b * n, out0 = (int64_t)(b + 1) * n;
  for (int32_t g = 0; g < p.ngroups; ++g) {
    const int K = p.gk[g], G = p.gg[g];
    const int32_t anchor = (int32_t)(out0 + p.col[(size_t)g * p.gmax]);
    for (int t = 0; t < K; ++t) uf.unite(anchor, (int32_t)(in0 + p.src[(size_t)g * p.kmax + t]));
    for (int q = 1; q < G; ++q) uf.unite(anchor, (int32_t)(out0 + p.col[(size_t)g * p.gmax + q]));
  }
}

// every component has <= cap nodes on each of the boundaries 0..m
bool within_cap(UF &uf, int32_t n, int m, int cap, std::vector<int32_t> &cnt,
                std::vector<int32_t> &stamp) {
  for (int b = 0; b <= m; ++b) {
    const int32_t tag = b + 1;
    for (int32_t i = 0; i < n; ++i) {
      const int32_t r = uf.find((int32_t)((int64_t)b * n + i));
      if (stamp[r] != tag) {
        stamp[r] = tag;
        cnt[r] = 0;
      }
      if (++cnt[r] > cap) return false;
    }
  }
  return true;
}

// first-fit-decreasing of the sub-component sizes of every full component into
// bins of `cap_cta` slots; returns the largest bin count (0 if a sub-component
// alone exceeds a bin)
int bins_needed(UF &full, UF &sub, int32_t n, int cap_cta, std::vector<int32_t> &size,
                std::vector<int32_t> &owner) {
  // size[sub root] = rows at boundary 0; owner[] lists sub roots per full root
  std::vector<std::pair<int32_t, int32_t>> roots;      // (full root, sub root)
  for (int32_t i = 0; i < n; ++i) {
    const int32_t sr = sub.find(i);
    if (size[sr]++ == 0) roots.push_back({full.find(i), sr});
  }
  std::sort(roots.begin(), roots.end(), [&](const auto &x, const auto &y) {
    return x.first != y.first ? x.first < y.first : size[x.second] > size[y.second];
  });
  int worst = 1;
  std::vector<int32_t> bins;
  for (size_t q = 0; q < roots.size();) {
    size_t e = q;
    bins.clear();
    while (e < roots.size() && roots[e].first == roots[q].first) {
      const int32_t sz = size[roots[e].second];
      if (sz > cap_cta) worst = 0;
      bool placed = false;
      for (auto &b : bins)
        if (b + sz <= cap_cta) {
          b += sz;
          placed = true;
          break;
        }
      if (!placed) bins.push_back(sz);
      ++e;
    }
    if (worst) worst = std::max<int>(worst, (int)bins.size());
    q = e;
  }
  for (auto &r : roots) size[r.second] = 0;
  (void)owner;
  return worst;
}

}  // namespace

// slots per CTA of a fused pass: 512 (row-major activations: 32-position
// tiles of 128 B row segments) or 1024 (position-blocked activations, where a
// CTA's rows are consecutive storage rows and 16-position tiles stay cheap);
// SDNN_PASS_CTA_ROWS = 128 / 256 / 512 / 1024 overrides for A/B runs.  A
// component larger than this spreads over a cluster of up to kMaxPassCluster CTAs
int pass_cta_rows(bool blocked) {
  static const int env = [] {
    const char *e = getenv("SDNN_PASS_CTA_ROWS");
    const int v = e ? atoi(e) : 0;
    return (v == 128 || v == 256 || v == 512 || v == 1024) ? v : 0;
  }();
  return env ? env : (blocked ? kMaxPassRows : kDefaultCtaRows);
}

// A pass [a, a+m) keeps every layer but the last inside one CTA: the
// sub-components of layers a..a+m-2 must fit pass_cta_rows() slots.  The last
// layer may read across a cluster of up to kMaxPassCluster CTAs, so the
// sub-components of a full component are bin-packed into at most
// cap / pass_cta_rows() CTAs (cap <= pass_cta_rows(): one CTA of cap slots).
namespace {
// longest feasible pass starting at layer a (1 = a plain layer) and, for every
// length k <= that, the largest component (rows at the first boundary); every
// prefix of a feasible pass is feasible
int max_pass_len(const std::vector<const PackedLayer *> &layers, int32_t n, int a, int cap,
                 int max_m, int cta_rows, std::vector<int> &rows_at, bool general) {
  const int L = (int)layers.size();
  rows_at.assign(max_m + 1, 1);
  if (!(cap > 0 && max_m > 1 && fusable(*layers[a], general))) return 1;
  const int cap_cta = std::min(cap, cta_rows);
  const int max_bins = std::max(1, cap / cta_rows);
  UF full, sub;
  std::vector<int32_t> cnt, stamp, size, owner, big(n);
  const int64_t nodes = (int64_t)(max_m + 1) * n;
  full.init(nodes);
  sub.init(nodes);
  cnt.assign(nodes, 0);
  stamp.assign(nodes, 0);
  size.assign(nodes, 0);
  add_layer(full, *layers[a], n, 0);
  auto largest = [&]() {
    std::fill(big.begin(), big.end(), 0);
    int mx = 0;
    for (int32_t i = 0; i < n; ++i) mx = std::max(mx, ++big[full.find(i)]);
    return mx;
  };
  rows_at[1] = 32;
  int m = 1;
  while (a + m < L && m < max_m && fusable(*layers[a + m], general) && inplace(*layers[a + m - 1])) {
    add_layer(sub, *layers[a + m - 1], n, m - 1);
    add_layer(full, *layers[a + m], n, m);
    std::fill(stamp.begin(), stamp.begin() + (int64_t)(m + 1) * n, 0);
    if (!within_cap(sub, n, m, cap_cta, cnt, stamp)) break;
    const int nb = bins_needed(full, sub, n, cap_cta, size, owner);
    if (nb == 0 || nb > max_bins) break;
    ++m;
    rows_at[m] = largest();
  }
  return m;
}

bool cost_planner() {                            // default; SDNN_PLAN=greedy for the greedy cover
  const char *e = getenv("SDNN_PLAN");
  return !(e && std::strcmp(e, "greedy") == 0);
}
}  // namespace

static std::vector<Step> plan_steps_greedy(const std::vector<const PackedLayer *> &layers, int32_t n,
                                           int cap, int max_m, int cta_rows, int a_begin, bool general) {
  std::vector<Step> steps;
  const int L = (int)layers.size();
  max_m = std::max(1, std::min(max_m, kMaxPassLayers));
  cap = std::min(cap, cta_rows * kMaxPassCluster);
  const int cap_cta = std::min(cap, cta_rows);
  const int max_bins = std::max(1, cap / cta_rows);
  UF full, sub;
  std::vector<int32_t> cnt, stamp, size, owner;
  for (int a = a_begin; a < L;) {
    int m = 1;
    if (cap > 0 && max_m > 1 && fusable(*layers[a], general)) {
      const int64_t nodes = (int64_t)(max_m + 1) * n;
      full.init(nodes);
      sub.init(nodes);
      cnt.assign(nodes, 0);
      stamp.assign(nodes, 0);
      size.assign(nodes, 0);
      add_layer(full, *layers[a], n, 0);
      // layer a+m-1 stops being the last layer of the pass: it must allow in-place slots
      while (a + m < L && m < max_m && fusable(*layers[a + m], general) && inplace(*layers[a + m - 1])) {
        add_layer(sub, *layers[a + m - 1], n, m - 1);
        add_layer(full, *layers[a + m], n, m);
        std::fill(stamp.begin(), stamp.end(), 0);
        if (!within_cap(sub, n, m, cap_cta, cnt, stamp)) break;
        const int nb = bins_needed(full, sub, n, cap_cta, size, owner);
        if (nb == 0 || nb > max_bins) break;
        ++m;
      }
    }
    Step s;
    s.a = a;
    s.m = m;
    steps.push_back(s);
    a += m;
  }
  return steps;
}

// The default cover (SDNN_PLAN=greedy: always the longest pass) -- the longest
// pass from every start layer (in parallel), then a shortest path over layer
// boundaries with a per-pass cost of 1 (one HBM round trip of the live rows)
// plus 0.3 for components above 512 rows (16-position tiles: measured 3.39 vs
// 2.61 ms on C4); ties go to the longer first pass.  Measured: C4 2021 vs
// 2056 ms/step, C3 368 vs 376 ms for the greedy cover.
static std::vector<Step> plan_steps_cost(const std::vector<const PackedLayer *> &layers, int32_t n,
                                         int cap, int max_m, int cta_rows, int a_begin, bool general) {
  const int L = (int)layers.size();
  std::vector<int> mm(L, 1);
  std::vector<std::vector<int>> rows(L);
  {
    std::atomic<int> next{a_begin};
    const int nt = std::max(1, std::min<int>((int)std::thread::hardware_concurrency(), 8));
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t)
      th.emplace_back([&] {
        for (int a = next++; a < L; a = next++) mm[a] = max_pass_len(layers, n, a, cap, max_m, cta_rows, rows[a], general);
      });
    for (auto &x : th) x.join();
  }
  // SDNN_PLAN_COST="big,small": penalties for >512-row components and for
  // 2-layer passes of <= 256 rows (A/B knobs; defaults 0.3, 0)
  double big = 0.3, small = 0.0;
  if (const char *e = getenv("SDNN_PLAN_COST")) sscanf(e, "%lf,%lf", &big, &small);
  std::vector<double> best(L + 1, 0.0);
  std::vector<int> choice(L + 1, 1);
  for (int a = L - 1; a >= a_begin; --a) {
    best[a] = 1e300;
    for (int k = std::min(mm[a], L - a); k >= 1; --k) {
      const double c = 1.0 + (k > 1 && rows[a][k] > 512 ? big : 0.0) +
                       (k == 2 && rows[a][k] <= 256 ? small : 0.0) + best[a + k];
      if (c < best[a] - 1e-9) {
        best[a] = c;
        choice[a] = k;
      }
    }
  }
  std::vector<Step> steps;
  for (int a = a_begin; a < L;) {
    Step s;
    s.a = a;
    s.m = choice[a];
    steps.push_back(s);
    a += s.m;
  }
  return steps;
}

std::vector<Step> plan_steps(const std::vector<const PackedLayer *> &layers, int32_t n, int cap,
                             int max_m, int cta_rows, int a_begin, bool general) {
  if (a_begin >= (int)layers.size()) return {};
  const int mm_ = std::max(1, std::min(max_m, kMaxPassLayers));
  const int cap_ = std::min(cap, cta_rows * kMaxPassCluster);
  return cost_planner() ? plan_steps_cost(layers, n, cap_, mm_, cta_rows, a_begin, general)
                        : plan_steps_greedy(layers, n, cap, max_m, cta_rows, a_begin, general);
}

static void build_pass_impl(const std::vector<const PackedLayer *> &layers, int32_t n, const Step &s,
                            int tile_floats, int cta_rows, PassHost &out, bool allow_dedup,
                            bool allow_vt = true, bool blocked = false, const Step *prev = nullptr);

void build_pass(const std::vector<const PackedLayer *> &layers, int32_t n, const Step &s,
                int tile_floats, int cta_rows, PassHost &out, bool share_values, bool blocked,
                const Step *prev) {
  build_pass_impl(layers, n, s, tile_floats, cta_rows, out, share_values, true, blocked, prev);
}

static void build_pass_impl(const std::vector<const PackedLayer *> &layers, int32_t n, const Step &s,
                            int tile_floats, int cta_rows, PassHost &out, bool allow_dedup, bool allow_vt,
                            bool blocked, const Step *prev) {
  const int m = s.m;
  UF full, sub;
  full.init((int64_t)(m + 1) * n);
  sub.init((int64_t)(m + 1) * n);
  for (int b = 0; b < m; ++b) add_layer(full, *layers[s.a + b], n, b);
  for (int b = 0; b + 1 < m; ++b) add_layer(sub, *layers[s.a + b], n, b);
  // components that own at least one group (have outputs); dense ids
  std::vector<int32_t> comp_of_root((size_t)(m + 1) * n, -1);
  int ncomp = 0;
  for (int b = 0; b < m; ++b) {
    const PackedLayer &p = *layers[s.a + b];
    for (int32_t g = 0; g < p.ngroups; ++g) {
      const int32_t r = full.find((int32_t)((int64_t)(b + 1) * n + p.col[(size_t)g * p.gmax]));
      if (comp_of_root[r] < 0) comp_of_root[r] = ncomp++;
    }
  }
  // boundary-0 rows of each component, grouped by sub-component, bin-packed
  // (first fit decreasing) into CTAs of pass_cta_rows() slots
  std::vector<std::vector<std::vector<int32_t>>> subs(ncomp);   // [comp][sub] rows
  {
    std::vector<int32_t> sub_idx((size_t)(m + 1) * n, -1);
    for (int32_t i = 0; i < n; ++i) {
      const int32_t c = comp_of_root[full.find(i)];
      if (c < 0) continue;                        // input neuron feeding nothing in this pass
      const int32_t sr = sub.find(i);
      if (sub_idx[sr] < 0) {
        sub_idx[sr] = (int32_t)subs[c].size();
        subs[c].emplace_back();
      }
      subs[c][sub_idx[sr]].push_back(i);
    }
  }
  std::vector<int32_t> prev_group;               // group of each neuron in layer a-1
  if (s.a > 0) {
    const PackedLayer &pp = *layers[s.a - 1];
    prev_group.assign(n, -1);
    for (int32_t g = 0; g < pp.ngroups; ++g)
      for (int u = 0; u < pp.gg[g]; ++u) prev_group[pp.col[(size_t)g * pp.gmax + u]] = g;
  }
  // writer component of each input row: the component (over the previous
  // step's layers) whose last layer writes it.  One item of the previous pass
  // stores all rows of its component for one tile, so rows of one writer
  // component placed next to each other make its stores runs of consecutive
  // storage rows (SDNN_PASS_WKEY=0: group order only)
  std::vector<int32_t> wroot;
  static const bool wkey_env = [] {
    const char *e = getenv("SDNN_PASS_WKEY");
    return !(e && atoi(e) == 0);
  }();
  if (wkey_env && prev && prev->m >= 1 && prev->a + prev->m == s.a) {
    UF w;
    w.init((int64_t)(prev->m + 1) * n);
    for (int b = 0; b < prev->m; ++b) add_layer(w, *layers[prev->a + b], n, b);
    wroot.assign(n, 0);
    for (int32_t x = 0; x < n; ++x) wroot[x] = w.find((int32_t)((int64_t)prev->m * n + x));
  }
  std::vector<std::vector<std::vector<int32_t>>> bins(ncomp);   // [comp][bin] rows
  int C = 1, R = 1;
  bool gen_pass = false;                          // per-slot weights somewhere in the pass
  for (int b = 0; b < m; ++b) gen_pass = gen_pass || !layers[s.a + b]->uniform;
  if (blocked && pass_wide_mode() == 2 && m >= 3 && !gen_pass) cta_rows = std::min(cta_rows, 512);   // 2-CTA clusters
  for (int c = 0; c < ncomp; ++c) {
    auto &v = subs[c];
    std::stable_sort(v.begin(), v.end(), [](const auto &x, const auto &y) { return x.size() > y.size(); });
    for (auto &sv : v) {
      bool placed = false;
      for (auto &b : bins[c])
        if ((int)(b.size() + sv.size()) <= cta_rows) {
          b.insert(b.end(), sv.begin(), sv.end());
          placed = true;
          break;
        }
      if (!placed) bins[c].push_back(sv);
    }
    for (auto &b : bins[c]) {
      // slot order: rows written by the same group of the previous layer
      // (layer a-1, the last layer of the previous pass) next to each other,
      // then ascending neuron id.  Any order is correct; with position-blocked
      // activations (make_plan) slots are consecutive storage rows, so a writer
      // group's member stores become runs of consecutive rows.
      if (prev_group.empty()) {
        std::sort(b.begin(), b.end());
      } else {
        std::sort(b.begin(), b.end(), [&](int32_t x, int32_t y) {
          if (!wroot.empty() && wroot[x] != wroot[y]) return wroot[x] < wroot[y];
          return prev_group[x] != prev_group[y] ? prev_group[x] < prev_group[y] : x < y;
        });
      }
      R = std::max<int>(R, (int)b.size());
    }
    C = std::max<int>(C, (int)bins[c].size());
  }
  // a component that needs more CTAs than a cluster holds is not buildable:
  // leave `out` empty (m = 0) and let plan_passes fall back (one-layer steps
  // run as plain layers, longer passes lose their last layer)
  out = PassHost();
  if (C > kMaxPassCluster) return;
  if (C > 1) C = C <= 2 ? 2 : 4;                  // cluster sizes 2 / 4
  {
    int Rp = 32;
    while (Rp < R) Rp <<= 1;
    if (!pass_variant(std::max(16, std::min(512, tile_floats / Rp)), C, 1)) return;   // no kernel instance
  }
  // slot code of a boundary node: (bin << 8) | slot within the bin
  std::vector<int32_t> slot((size_t)(m + 1) * n, -1);
  std::vector<int32_t> bin_of_sub((size_t)(m + 1) * n, 0);
  out.a = s.a;
  out.m = m;
  out.ncomp = ncomp;
  out.C = C;
  out.R = R;
  out.rin = R;
  int Rp = 32;                                    // one tile of tile_floats per CTA
  while (Rp < R) Rp <<= 1;
  out.T = std::max(16, std::min(512, tile_floats / Rp));
  out.NB = 1;
  // 513-1024 rows in one CTA (position-blocked plans): 32-position tiles in
  // rotating halves, one CTA per SM (pass_wide.cu) instead of 16-position tiles
  if (pass_wide_enabled() && blocked && C == 1 && Rp == 1024) {
    out.T = 32;
    out.NB = 3;
  }
  // <= 512 rows (SDNN_PASS_T32=1: <= 256) in the blocked layout: CTAs of
  // ceil(rows / 128) warps with S 32-position tiles (k_pass_t32)
  if (out.NB == 1 && C == 1 && blocked && pass_t32_mode() > 0 && Rp <= (pass_t32_mode() >= 2 ? 512 : 256)) {
    out.T = 32;
    out.NW = Rp <= 128 ? 1 : Rp <= 256 ? 2 : 4;
    out.S = pass_t32_stages(out.NW);
    if (!pass_t32_variant(out.NW, out.S)) out.NW = 0;
  }
  // per-slot-weight layers in the pass: only k_pass_gw runs them (blocked
  // layout, one CTA per component of <= 512 rows); anything else is not
  // buildable here and plan_passes falls back (shorter pass / plain layer)
  if (gen_pass) {
    if (!(blocked && C == 1 && Rp <= 1024)) {
      out = PassHost();
      return;
    }
    out.general = true;
    out.T = 32;
    out.NB = 1;
    out.NW = Rp <= 128 ? 4 : 8;                   // warps: one group (32 rows) per warp and round
    out.S = 1;
    out.split.clear();
  }
  // SDNN_PASS_WIDE=2: components of 513-1024 rows (up to 2048 with
  // fuse_rows = 2048) over 2- (4-) CTA clusters of k_pass_t32 (512 rows per
  // CTA, binned with cta = 512 above)
  if (out.NB == 1 && (C == 2 || C == 4) && R <= 512 && blocked && pass_wide_mode() == 2 &&
      pass_t32_variant(4, 1, C)) {
    out.T = 32;
    out.NW = 4;
    out.S = 1;
  }
  if (out.NB == 3) {                              // half 0 = the first 512 slots
    out.split.assign(ncomp, 0);
    for (int c = 0; c < ncomp; ++c) out.split[c] = std::min<int>(512, (int)bins[c][0].size());
  }
  // Bank-parity slot order for 16-position tiles (k_pass<16>: 64 B rows, two
  // per 128 B shared-memory line).  A quarter-warp phase of k_pass<16> holds the
  // units of groups 2i and 2i+1 (record order) at the same term t: their rows
  // src_2i[t] and src_2i+1[t] conflict when their slots have equal parity, and
  // so do the in-place member stores (member v goes to the slot of source v).
  // Any slot order and any member -> source-slot assignment within a group is
  // correct, so the planner chooses them: at boundary 0 the parity of a row is
  // its slot position's; at boundary j >= 1 a member takes the parity of the
  // source slot of its group (layer j-1) it is assigned to.  Per boundary, each
  // read pair (x, y) wants opposite parities, each writer (the slot order /
  // layer j-1 group) has a fixed number of even slots, and, when layer j writes
  // in place, each group of layer j wants half of its slots even (so the next
  // boundary stays solvable): an orientation problem, solved by local search
  // (an Eulerian orientation satisfies the writer counts alone).  On C4 it cuts
  // the equal-parity read pairs of these passes from ~50 % to < 1 %, but the
  // passes read 18.4 instead of 14.6 GB from DRAM and the step slowed down
  // (2000 vs 1929 ms/step with SDNN_PASS_WIDE=0), so it is opt-in
  // (SDNN_PASS_PARITY=1).  member_at[b][g * gmax + v] = member written into the
  // slot of source v of group g of layer b.
  std::vector<std::vector<int32_t>> member_at(m);
  static const bool parity_env = [] {            // opt-in (measured slower, see below)
    const char *e = getenv("SDNN_PASS_PARITY");
    return e && atoi(e) == 1;
  }();
  static const bool vt_env0 = [] {
    const char *e = getenv("SDNN_PASS_VT");
    return e && atoi(e) == 1;
  }();
  if (parity_env && out.T == 16 && C == 1 && out.NB == 1 && !allow_dedup && !vt_env0) {
    for (int b = 0; b + 1 < m; ++b) {
      const PackedLayer &p = *layers[s.a + b];
      member_at[b].assign(p.col.begin(), p.col.end());
    }
    // groups of each layer per component, ascending (the record order)
    std::vector<std::vector<std::vector<int32_t>>> cg(m, std::vector<std::vector<int32_t>>(ncomp));
    for (int b = 0; b < m; ++b) {
      const PackedLayer &p = *layers[s.a + b];
      for (int32_t g = 0; g < p.ngroups; ++g) {
        const int32_t c = comp_of_root[full.find((int32_t)((int64_t)(b + 1) * n + p.col[(size_t)g * p.gmax]))];
        if (c >= 0) cg[b][c].push_back(g);
      }
    }
    std::vector<int8_t> parP(n, 0), par(n, 0);   // parities at boundaries b-1 and b (this component)
    std::vector<int32_t> wof(n, -1);             // writer index of a node
    std::vector<int32_t> eidx(n, -1);            // edge of a node
    uint64_t rng = 0x9E3779B97F4A7C15ull ^ (uint64_t)s.a;
    auto rnd = [&]() {
      rng ^= rng << 13;
      rng ^= rng >> 7;
      rng ^= rng << 17;
      return rng;
    };
    for (int c = 0; c < ncomp; ++c) {
      std::vector<int32_t> &rows0 = bins[c][0];
      for (int b = 0; b < m; ++b) {
        const PackedLayer &p = *layers[s.a + b];
        const auto &G = cg[b][c];
        // nodes of boundary b with their writer: b = 0 the slot order (writer 0),
        // else the layer b-1 group that has them as a member
        std::vector<int32_t> nodes;
        std::vector<int32_t> cap;                  // even slots per writer
        std::vector<std::vector<int32_t>> wsrc;    // b >= 1: source-slot parities per writer
        if (b == 0) {
          nodes = rows0;
          cap.push_back(((int)nodes.size() + 1) / 2);
          for (int32_t x : nodes) wof[x] = 0;
        } else {
          const PackedLayer &pp = *layers[s.a + b - 1];
          const auto &W = cg[b - 1][c];
          for (size_t w = 0; w < W.size(); ++w) {
            const int32_t g = W[w];
            int e = 0;
            for (int v = 0; v < pp.gg[g]; ++v) {
              const int32_t x = pp.col[(size_t)g * pp.gmax + v];
              nodes.push_back(x);
              wof[x] = (int32_t)w;
            }
            for (int v = 0; v < pp.gg[g]; ++v) e += parP[pp.src[(size_t)g * pp.kmax + v]] == 0;
            cap.push_back(e);
          }
        }
        // read pairs of layer b (groups 2i, 2i+1 of the record, the same term)
        std::vector<std::array<int32_t, 2>> E;
        std::vector<int32_t> epair;                // reader pair of each edge
        for (size_t i = 0; i + 1 < G.size(); i += 2) {
          const int32_t ga = G[i], gb = G[i + 1];
          const int kk = std::min(p.gk[ga], p.gk[gb]);
          for (int t = 0; t < kk; ++t) {
            const int32_t x = p.src[(size_t)ga * p.kmax + t], y = p.src[(size_t)gb * p.kmax + t];
            if (wof[x] < 0 || wof[y] < 0) continue;   // (a node without a writer: free)
            eidx[x] = eidx[y] = (int32_t)E.size();
            E.push_back({x, y});
            epair.push_back((int32_t)(i / 2));
          }
        }
        // balance of layer b's groups (writers of boundary b+1) when in place:
        // group 2i gets half of its first gg sources even
        const bool bal = b + 1 < m;
        const int npairs = (int)G.size() / 2;
        std::vector<int32_t> half(npairs, 0);
        for (int i = 0; i < npairs; ++i) half[i] = p.gg[G[2 * i]] / 2;
        std::vector<int8_t> o(E.size());           // orientation: 0 = x even, 1 = y even
        std::vector<int32_t> cw(cap.size(), 0), cr(npairs, 0);
        auto ga_counts = [&](size_t e) {           // edge e counts for group 2i's balance
          const int32_t ga = G[2 * epair[e]];
          const int t = (int)(e - (size_t)(std::lower_bound(epair.begin(), epair.end(), epair[e]) - epair.begin()));
          return t < p.gg[ga];
        };
        std::vector<int8_t> inbal(E.size());
        for (size_t e = 0; e < E.size(); ++e) {
          o[e] = (int8_t)(e & 1);
          inbal[e] = bal && ga_counts(e);
          cw[wof[E[e][o[e]]]]++;
          if (inbal[e] && o[e] == 0) cr[epair[e]]++;
        }
        auto cost_w = [&](int w, int d) { return std::abs(cw[w] + d - cap[w]) - std::abs(cw[w] - cap[w]); };
        auto cost_r = [&](int i, int d) { return std::abs(cr[i] + d - half[i]) - std::abs(cr[i] - half[i]); };
        for (int it = 0; it < 60 && !E.empty(); ++it) {
          int64_t bad = 0;
          for (size_t w = 0; w < cap.size(); ++w) bad += std::abs(cw[w] - cap[w]);
          if (bal)
            for (int i = 0; i < npairs; ++i) bad += std::abs(cr[i] - half[i]);
          if (bad == 0) break;
          for (size_t q = 0; q < E.size(); ++q) {
            const size_t e = rnd() % E.size();
            const int wold = wof[E[e][o[e]]], wnew = wof[E[e][1 - o[e]]];
            int d = wold == wnew ? 0 : cost_w(wold, -1) + cost_w(wnew, +1);
            if (inbal[e]) d += cost_r(epair[e], o[e] == 0 ? -1 : +1);
            if (d < 0 || (d == 0 && (rnd() & 3) == 0)) {
              cw[wold]--;
              cw[wnew]++;
              if (inbal[e]) cr[epair[e]] += o[e] == 0 ? -1 : +1;
              o[e] ^= 1;
            }
          }
        }
        // wanted parity of every node (free nodes: -1), then exact writer counts
        std::vector<int8_t> want(nodes.size(), -1);
        for (size_t q = 0; q < nodes.size(); ++q) {
          const int32_t x = nodes[q];
          const int32_t e = eidx[x];
          if (e >= 0) want[q] = (int8_t)(E[e][o[e]] == x ? 0 : 1);
        }
        std::vector<std::vector<int32_t>> ev(cap.size()), od(cap.size()), fr(cap.size());
        for (size_t q = 0; q < nodes.size(); ++q)
          (want[q] == 0 ? ev : want[q] == 1 ? od : fr)[wof[nodes[q]]].push_back(nodes[q]);
        for (size_t w = 0; w < cap.size(); ++w) {
          auto &E0 = ev[w], &O0 = od[w], &F0 = fr[w];
          while ((int)E0.size() < cap[w] && !F0.empty()) { E0.push_back(F0.back()); F0.pop_back(); }
          while ((int)E0.size() < cap[w] && !O0.empty()) { E0.push_back(O0.back()); O0.pop_back(); }
          while ((int)E0.size() > cap[w]) { O0.push_back(E0.back()); E0.pop_back(); }
          for (int32_t x : F0) O0.push_back(x);
          for (int32_t x : E0) par[x] = 0;
          for (int32_t x : O0) par[x] = 1;
          if (b == 0) {                            // slot order: evens at even positions
            std::vector<int32_t> ord(nodes.size());
            size_t ie = 0, io = 0;
            for (size_t q = 0; q < ord.size(); ++q) ord[q] = (q & 1) ? O0[io++] : E0[ie++];
            rows0 = ord;
          } else {                                 // member -> source slot of matching parity
            const PackedLayer &pp = *layers[s.a + b - 1];
            const int32_t g = cg[b - 1][c][w];
            size_t ie = 0, io = 0;
            for (int v = 0; v < pp.gg[g]; ++v)
              member_at[b - 1][(size_t)g * pp.gmax + v] =
                  parP[pp.src[(size_t)g * pp.kmax + v]] == 0 ? E0[ie++] : O0[io++];
          }
        }
        for (int32_t x : nodes) {
          wof[x] = -1;
          eidx[x] = -1;
          parP[x] = par[x];                        // boundary b becomes the previous one
        }
      }
    }
  }
  out.in_rows.assign((size_t)ncomp * C * R, -1);
  out.in_count.assign((size_t)ncomp * C, 0);
  for (int c = 0; c < ncomp; ++c)
    for (int b = 0; b < (int)bins[c].size(); ++b) {
      const auto &rows = bins[c][b];
      for (size_t q = 0; q < rows.size(); ++q) {
        slot[rows[q]] = (b << 10) | (int32_t)q;
        bin_of_sub[sub.find(rows[q])] = b;
        out.in_rows[((size_t)c * C + b) * R + q] = rows[q];
      }
      out.in_count[(size_t)c * C + b] = (int32_t)rows.size();
    }
  out.layers.resize(m);
  // Value tables for the passes of 16-position tiles (1024-row components: two
  // 64 B rows share each 128 B shared-memory line, so two units of one
  // quarter-warp phase that read rows of equal parity conflict): when the
  // members of a group share one value (uniform weights, equal biases), a
  // non-last layer b writes it twice into line q of table b & 1 -- copy 0 in
  // the first 64 B, copy 1 in the second -- once every group has read its
  // sources; the next layer's terms read line g(t), the unit in the first half
  // of a phase copy 0 and the one in the second half copy 1, so every phase
  // covers both bank halves.  Opt-in (SDNN_PASS_VT=1): exact, and it removes
  // 91 % of the shared stores and a third of the load bank conflicts of these
  // passes, but the C4 step was measured slower (1977 vs 1934 ms/step; the
  // sampled pass read 10.4 instead of 7.6 GB from DRAM -- the two CTAs that
  // share each 128 B line of the half-row loads drift apart).
  static const bool vt_env = [] {
    const char *e = getenv("SDNN_PASS_VT");
    return e && atoi(e) == 1;
  }();
  bool vt = false;
  if (vt_env && allow_vt && m >= 2 && C == 1 && out.T == 16) {
    vt = true;
    for (int b = 0; b + 1 < m && vt; ++b) {
      const PackedLayer &p = *layers[s.a + b];
      bool eq = p.uniform && p.gmax > 1;
      for (int32_t j = 1; j < n && eq; ++j) eq = std::memcmp(&p.bias[j], &p.bias[0], 4) == 0;
      vt = eq;
    }
  }
  // value sharing (SDNN_F_SHARE_VALUES, opt-in): in a layer with uniform
  // weights whose member biases are all equal, every member of a group has
  // bit-identical outputs, so a non-last layer stores the group's value once --
  // into the slot of its source 0 when only this group reads it, else into a
  // slot no group of the layer reads -- and the next layer's terms read that
  // slot.  The chains are unchanged (same operands, same order); only the
  // shared-memory stores drop by the group size.  Measured on C4: 2021 vs 1945
  // ms/step (the 1024-row passes slow down: 3.92 vs 3.11 ms), so off by default.
  const bool dedup_on = allow_dedup && !vt && out.NB != 3 && out.NW == 0;   // (pass_wide.cu has no value slots)
  // A layer after a sharing layer reads shared slots, so it cannot overwrite its
  // sources in place: it must share too (or be the last layer) -- decided from
  // the back.
  std::vector<char> dedup(m, 0);
  for (int b = m - 2; b >= 0 && dedup_on; --b) {
    const PackedLayer &p = *layers[s.a + b];
    bool eq = p.uniform && p.gmax > 1;           // (groups of one member gain nothing)
    for (int32_t j = 1; j < n && eq; ++j) eq = std::memcmp(&p.bias[j], &p.bias[0], 4) == 0;
    dedup[b] = eq && (b + 1 == m - 1 || dedup[b + 1]);
  }
  for (int b = 0; b < m; ++b) {
    const PackedLayer &p = *layers[s.a + b];
    const bool last = b == m - 1;
    // groups of each (component, bin): non-last layers by their sub-component's
    // bin (all sources local), the last layer round robin over the bins
    std::vector<std::vector<int32_t>> groups((size_t)ncomp * C);
    std::vector<int32_t> rr(ncomp, 0);
    for (int32_t g = 0; g < p.ngroups; ++g) {
      const int32_t node = (int32_t)((int64_t)(b + 1) * n + p.col[(size_t)g * p.gmax]);
      const int32_t c = comp_of_root[full.find(node)];
      const int bin = last ? (rr[c]++ % C) : bin_of_sub[sub.find(node)];
      groups[(size_t)c * C + bin].push_back(g);
    }
    int NG = 1;
    for (auto &v : groups) NG = std::max<int>(NG, (int)v.size());
    PassHostLayer &H = out.layers[b];
    H.NG = NG;
    H.wu = p.wu;
    H.dedup = dedup[b];
    if (vt && NG > 32) {                           // one round of units per layer (4 warps x 8 units),
                                                   // so the table stores follow every read of the tile
      build_pass_impl(layers, n, s, tile_floats, cta_rows, out, allow_dedup, false, blocked, prev);
      return;
    }
    // layer b (non-last) writes table b & 1 (lines 0.. or 256..), layer b > 0 reads table (b-1) & 1
    H.vt = vt ? ((last ? 0 : 1 | ((b & 1) << 2)) | (b > 0 ? 2 : 0)) : 0;
    const size_t units = (size_t)ncomp * C;
    H.src.assign(units * NG * 32, 0);
    H.bias.assign(units * NG * 32, 0.f);
    H.k.assign(units * NG, 0);
    H.g.assign(units * NG, 0);
    H.general = !p.uniform;
    if (H.general) H.gid.assign(units * NG, 0);
    if (last) H.orow.assign(units * NG * 32, 0);      // u16: N <= 65536
    const int64_t in0 = (int64_t)b * n, out0 = (int64_t)(b + 1) * n;
    if (!last && dedup[b]) H.vs.assign(units * NG, 0);
    // the input slots of this layer are exclusive to one group each unless the
    // previous layer shared values (then several groups read one value slot)
    const bool excl = b == 0 || !dedup[b - 1];
    std::vector<char> live;
    for (size_t cb = 0; cb < units; ++cb) {
      if (!last && dedup[b] && !excl) live.assign(kMaxPassRows, 0);
      std::vector<int32_t> code0(groups[cb].size());
      for (size_t q = 0; q < groups[cb].size(); ++q) {
        const int32_t g = groups[cb][q];
        const size_t rec = cb * NG + q;
        const int K = p.gk[g], G = p.gg[g];
        H.k[rec] = (uint8_t)K;
        H.g[rec] = (uint8_t)G;
        if (!p.uniform) H.gid[rec] = (uint16_t)g;      // per-slot weights: W_l[g] (k_pass_gw)
        // keeps the ascending source order (canonical chain); non-last layers read
        // their own CTA's slots, the last layer the (bin << 10 | slot) code
        int32_t code[32];
        for (int t = 0; t < K; ++t) {
          code[t] = slot[in0 + p.src[(size_t)g * p.kmax + t]];
          H.src[rec * 32 + t] = (uint16_t)(last ? code[t] : (code[t] & 0x3ff));
          if (!live.empty()) live[code[t] & 0x3ff] = 1;
        }
        code0[q] = K > 0 ? code[0] : 0;
        for (int u = 0; u < G; ++u) {
          const int32_t j = (!last && !member_at[b].empty()) ? member_at[b][(size_t)g * p.gmax + u]
                                                             : p.col[(size_t)g * p.gmax + u];
          H.bias[rec * 32 + u] = p.bias[j];
          if (last)
            H.orow[rec * 32 + u] = (uint16_t)j;
          else if (vt)                       // value table b & 1: line = record index q
            slot[out0 + j] = (b & 1) * 256 + (int32_t)q;
          else if (!dedup[b])                // member u overwrites the slot of source u
            slot[out0 + j] = code[u];
        }
      }
      if (last || !dedup[b]) continue;
      // shared values: one slot per group -- its own source-0 slot when the
      // inputs are exclusive, else a slot no group of this layer reads
      int32_t next_free = 0;
      for (size_t q = 0; q < groups[cb].size(); ++q) {
        const int32_t g = groups[cb][q];
        int32_t vcode = code0[q];
        if (!excl) {
          while (next_free < R && live[next_free]) ++next_free;
          if (next_free >= R) {                 // no free slot left: build without sharing
            build_pass_impl(layers, n, s, tile_floats, cta_rows, out, false, allow_vt, blocked, prev);
            return;
          }
          vcode = (code0[q] & ~0x3ff) | next_free;
          ++next_free;
        }
        H.vs[cb * NG + q] = (uint16_t)(vcode & 0x3ff);
        for (int u = 0; u < p.gg[g]; ++u) slot[out0 + p.col[(size_t)g * p.gmax + u]] = vcode;
      }
    }
  }
  // ---- per-(component, bin) records ----
  // a layer whose members all carry the same bias (bitwise) stores it once (bu)
  for (int b = 0; b < m; ++b) {
    PassHostLayer &H = out.layers[b];
    bool first = true, uni = true;
    uint32_t ref = 0;
    for (size_t r = 0; r < H.g.size() && uni; ++r)
      for (int u = 0; u < H.g[r]; ++u) {
        uint32_t bits;
        std::memcpy(&bits, &H.bias[r * 32 + u], 4);
        if (first) {
          ref = bits;
          first = false;
        } else if (bits != ref) {
          uni = false;
          break;
        }
      }
    H.bias_uniform = uni;
    std::memcpy(&H.bu, &ref, 4);
  }
  int32_t off = 0;
  for (int b = 0; b < m; ++b) {
    PassHostLayer &H = out.layers[b];
    H.off_kg = off;
    off += (H.NG * 2 + 15) / 16 * 16;
    H.off_src = off;
    off += H.NG * 64;
    H.off_gid = -1;
    if (H.general) {                              // group ids (u16) of a per-slot-weight layer
      H.off_gid = off;
      off += (H.NG * 2 + 15) / 16 * 16;
    }
    H.off_vs = -1;
    if (!H.vs.empty()) {                          // shared-value slots (dedup), u16 per group
      H.off_vs = off;
      off += (H.NG * 2 + 15) / 16 * 16;
    }
    H.off_bias = -1;
    if (!H.bias_uniform) {
      H.off_bias = off;
      off += H.NG * 128;
    }
    if (b == m - 1) {
      H.off_orow = off;
      off += H.NG * 64;
    }
  }
  out.rec_bytes = off;
  if (getenv("SDNN_PLAN_DEBUG")) {
    // 16-position tiles: read pairs (groups 2i, 2i+1, same term) whose slots
    // have equal parity (one shared-memory bank conflict each), per layer
    std::string conf;
    if (out.T == 16 && C == 1)
      for (int b = 0; b < m; ++b) {
        const PassHostLayer &H = out.layers[b];
        int64_t cnt = 0, tot = 0;
        for (size_t cb = 0; cb < (size_t)ncomp; ++cb)
          for (int q = 0; q + 1 < H.NG; q += 2) {
            const int kk = std::min(H.k[cb * H.NG + q], H.k[cb * H.NG + q + 1]);
            for (int t = 0; t < kk; ++t) {
              tot++;
              cnt += ((H.src[(cb * H.NG + q) * 32 + t] ^ H.src[(cb * H.NG + q + 1) * 32 + t]) & 1) == 0;
            }
          }
        conf += " " + std::to_string(cnt) + "/" + std::to_string(tot);
      }
    fprintf(stderr, "pass a=%d m=%d R=%d T=%d C=%d NB=%d ncomp=%d rec=%d vt=%d/%d share=%d parity-conflicts%s\n", s.a,
            m, R, out.T, C, out.NB, ncomp, off, out.layers[0].vt, m > 1 ? out.layers[1].vt : -1, (int)allow_dedup,
            conf.c_str());
  }
  // components of <= 128 rows: two half-size tiles per CTA (double-buffered)
  // when both records fit and a kernel instance exists (SDNN_PASS_NB=1: off).
  // Measured on C4: 128-row passes 2.69 ms (T = 64 x 2) vs 2.75 ms (T = 128);
  // 256-row passes 2.90 ms (T = 32 x 2) vs 2.61 ms (T = 64), so not for those
  {
    static const bool nb2 = [] {
      const char *e = getenv("SDNN_PASS_NB");
      return !(e && atoi(e) == 1);
    }();
    const int T2 = std::max(16, std::min(512, tile_floats / 2 / Rp));
    if (nb2 && out.NW == 0 && C == 1 && Rp <= 128 && ncomp >= 256 && off <= ((kPassRecMax / 2) & ~15) &&
        pass_variant(T2, 1, 2)) {                 // (C2's 32-component passes: 18.8 vs 18.4 ms without)
      out.NB = 2;
      out.T = T2;
    }
  }
  const size_t units = (size_t)ncomp * C;
  out.rec.assign(units * off, 0);
  for (size_t cb = 0; cb < units; ++cb) {
    unsigned char *r = out.rec.data() + cb * off;
    for (int b = 0; b < m; ++b) {
      const PassHostLayer &H = out.layers[b];
      const size_t g0 = cb * H.NG;
      for (int q = 0; q < H.NG; ++q) {
        const uint16_t kg = (uint16_t)(H.k[g0 + q] | (H.g[g0 + q] << 8));
        std::memcpy(r + H.off_kg + 2 * q, &kg, 2);
      }
      std::memcpy(r + H.off_src, H.src.data() + g0 * 32, (size_t)H.NG * 64);
      if (H.off_vs >= 0) std::memcpy(r + H.off_vs, H.vs.data() + g0, (size_t)H.NG * 2);
      if (H.off_gid >= 0) std::memcpy(r + H.off_gid, H.gid.data() + g0, (size_t)H.NG * 2);
      if (H.off_bias >= 0) std::memcpy(r + H.off_bias, H.bias.data() + g0 * 32, (size_t)H.NG * 128);
      if (H.off_orow >= 0) std::memcpy(r + H.off_orow, H.orow.data() + g0 * 32, (size_t)H.NG * 64);
    }
  }
}

std::vector<Step> plan_passes(const std::vector<const PackedLayer *> &layers, int32_t n, int cap,
                              int max_m, int tile_floats, int threads,
                              std::vector<PassHost> *built, int cta_rows, bool single_passes,
                              bool share_values) {
  // per-slot-weight layers join passes in blocked plans (k_pass_gw) only on
  // request (SDNN_PASS_GENERAL=1): exact, but measured slower than the
  // single-layer k_layer_bulkw steps (C4-RW 10.9 vs 4.1 s/step, C3-RW 3.17 vs
  // 1.52 s: the weights of every term come from L2 into registers, 96-128
  // registers per thread, two CTAs per SM)
  static const bool gen_env = [] {
    const char *e = getenv("SDNN_PASS_GENERAL");
    return e && atoi(e) == 1;
  }();
  const bool general = single_passes && gen_env;
  std::vector<Step> steps = plan_steps(layers, n, cap, max_m, cta_rows, 0, general);
  std::vector<PassHost> ph(steps.size());
  std::vector<char> done(steps.size(), 0);
  // single_passes: a lone fusable layer also runs as a (one-layer) pass
  auto is_pass = [&](const Step &x) {
    return x.m > 1 || (single_passes && cap > 0 && fusable(*layers[x.a], general));
  };
  for (;;) {
    std::vector<int> todo;
    for (int i = 0; i < (int)steps.size(); ++i)
      if (is_pass(steps[i]) && !done[i]) todo.push_back(i);
    std::atomic<int> next{0};
    std::vector<std::thread> th;
    const int nt = std::max(1, std::min<int>(threads, (int)todo.size()));
    for (int t = 0; t < nt && !todo.empty(); ++t)
      th.emplace_back([&] {
        for (int q = next++; q < (int)todo.size(); q = next++)
          build_pass(layers, n, steps[todo[q]], tile_floats, cta_rows, ph[todo[q]], share_values, single_passes,
                     todo[q] > 0 ? &steps[todo[q] - 1] : nullptr);
      });
    for (auto &x : th) x.join();
    for (int i : todo) done[i] = 1;
    // the first pass whose record does not fit loses its last layer, and the
    // layers after it are planned again (any prefix of a pass is a pass)
    int bad = -1;
    for (int i = 0; i < (int)steps.size() && bad < 0; ++i)
      if (steps[i].m > 1 && (ph[i].m == 0 || ph[i].rec_bytes > kPassRecMax)) bad = i;
    for (int i = 0; i < (int)steps.size(); ++i)   // a one-layer record that does not fit: plain layer
      if (steps[i].m == 1 && ph[i].rec_bytes > kPassRecMax) ph[i] = PassHost();
    if (bad < 0) break;
    Step &S = steps[bad];
    S.m -= 1;
    const int resume = S.a + S.m;
    steps.resize(bad + 1);
    ph.resize(bad + 1);
    done.resize(bad + 1);
    done[bad] = 0;
    ph[bad] = PassHost();
    for (const Step &x : plan_steps(layers, n, cap, max_m, cta_rows, resume, general)) {
      steps.push_back(x);
      ph.emplace_back();
      done.push_back(0);
    }
  }
  if (built) built->swap(ph);
  return steps;
}

}  // namespace sdnn
