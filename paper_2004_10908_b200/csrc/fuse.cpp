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
#include <cmath>
#include <atomic>
#include <cstring>
#include <numeric>
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

bool fusable(const PackedLayer &p) { return p.uniform && p.kmax <= 32 && p.gmax <= 32; }

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

}  // namespace

std::vector<Step> plan_steps(const std::vector<const PackedLayer *> &layers, int32_t n, int cap,
                             int max_m) {
  std::vector<Step> steps;
  const int L = (int)layers.size();
  max_m = std::max(1, std::min(max_m, kMaxPassLayers));
  UF uf;
  std::vector<int32_t> cnt, stamp;
  for (int a = 0; a < L;) {
    int m = 1;
    if (cap > 0 && max_m > 1 && fusable(*layers[a])) {
      const int64_t nodes = (int64_t)(max_m + 1) * n;
      uf.init(nodes);
      cnt.assign(nodes, 0);
      stamp.assign(nodes, 0);
      add_layer(uf, *layers[a], n, 0);
      if (within_cap(uf, n, 1, cap, cnt, stamp)) {
        // layer a+m-1 stops being the last layer of the pass: it must allow in-place slots
        while (a + m < L && m < max_m && fusable(*layers[a + m]) && inplace(*layers[a + m - 1])) {
          add_layer(uf, *layers[a + m], n, m);
          std::fill(stamp.begin(), stamp.end(), 0);
          if (!within_cap(uf, n, m + 1, cap, cnt, stamp)) break;
          ++m;
        }
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

void build_pass(const std::vector<const PackedLayer *> &layers, int32_t n, const Step &s,
                int tile_floats, PassHost &out) {
  const int m = s.m;
  UF uf;
  uf.init((int64_t)(m + 1) * n);
  for (int b = 0; b < m; ++b) add_layer(uf, *layers[s.a + b], n, b);
  // components that own at least one group (have outputs); dense ids
  std::vector<int32_t> comp_of_root((size_t)(m + 1) * n, -1);
  int ncomp = 0;
  for (int b = 0; b < m; ++b) {
    const PackedLayer &p = *layers[s.a + b];
    for (int32_t g = 0; g < p.ngroups; ++g) {
      const int32_t r = uf.find((int32_t)((int64_t)(b + 1) * n + p.col[(size_t)g * p.gmax]));
      if (comp_of_root[r] < 0) comp_of_root[r] = ncomp++;
    }
  }
  // boundary-0 rows of each component -> smem slots 0..cnt-1 (ascending neuron id)
  std::vector<int32_t> slot((size_t)(m + 1) * n, -1);
  std::vector<std::vector<int32_t>> rows_in(ncomp);
  for (int32_t i = 0; i < n; ++i) {
    const int32_t c = comp_of_root[uf.find(i)];
    if (c < 0) continue;                          // input neuron feeding nothing in this pass
    slot[i] = (int32_t)rows_in[c].size();
    rows_in[c].push_back(i);
  }
  out = PassHost();
  out.a = s.a;
  out.m = m;
  out.ncomp = ncomp;
  int R = 1;
  for (auto &v : rows_in) R = std::max<int>(R, (int)v.size());
  out.R = R;
  out.rin = R;
  int T = 512;                                    // one tile of tile_floats per component
  while (T > 128 && (int64_t)R * T > tile_floats) T >>= 1;
  out.T = T;
  out.in_rows.assign((size_t)ncomp * R, -1);
  out.in_count.assign(ncomp, 0);
  for (int c = 0; c < ncomp; ++c) {
    std::copy(rows_in[c].begin(), rows_in[c].end(), out.in_rows.begin() + (size_t)c * R);
    out.in_count[c] = (int32_t)rows_in[c].size();
  }
  out.layers.resize(m);
  for (int b = 0; b < m; ++b) {
    const PackedLayer &p = *layers[s.a + b];
    const bool last = b == m - 1;
    std::vector<std::vector<int32_t>> groups(ncomp);
    for (int32_t g = 0; g < p.ngroups; ++g) {
      const int32_t c =
          comp_of_root[uf.find((int32_t)((int64_t)(b + 1) * n + p.col[(size_t)g * p.gmax]))];
      groups[c].push_back(g);
    }
    int NG = 1;
    for (auto &v : groups) NG = std::max<int>(NG, (int)v.size());
    PassHostLayer &H = out.layers[b];
    H.NG = NG;
    H.wu = p.wu;
    H.src.assign((size_t)ncomp * NG * 32, 0);
    H.bias.assign((size_t)ncomp * NG * 32, 0.f);
    H.k.assign((size_t)ncomp * NG, 0);
    H.g.assign((size_t)ncomp * NG, 0);
    if (last) H.orow.assign((size_t)ncomp * NG * 32, 0);
    const int64_t in0 = (int64_t)b * n, out0 = (int64_t)(b + 1) * n;
    for (int c = 0; c < ncomp; ++c)
      for (size_t q = 0; q < groups[c].size(); ++q) {
        const int32_t g = groups[c][q];
        const size_t rec = (size_t)c * NG + q;
        const int K = p.gk[g], G = p.gg[g];
        H.k[rec] = (uint8_t)K;
        H.g[rec] = (uint8_t)G;
        for (int t = 0; t < K; ++t)        // keeps the ascending source order (canonical chain)
          H.src[rec * 32 + t] = (uint16_t)slot[in0 + p.src[(size_t)g * p.kmax + t]];
        for (int u = 0; u < G; ++u) {
          const int32_t j = p.col[(size_t)g * p.gmax + u];
          H.bias[rec * 32 + u] = p.bias[j];
          if (last)
            H.orow[rec * 32 + u] = j;
          else                             // member u overwrites the slot of source u
            slot[out0 + j] = H.src[rec * 32 + u];
        }
      }
  }
  // ---- per-component records ----
  int32_t off = 0;
  for (int b = 0; b < m; ++b) {
    PassHostLayer &H = out.layers[b];
    H.off_kg = off;
    off += (H.NG * 2 + 15) / 16 * 16;
    H.off_src = off;
    off += H.NG * 64;
    H.off_bias = off;
    off += H.NG * 128;
    if (b == m - 1) {
      H.off_orow = off;
      off += H.NG * 128;
    }
  }
  out.rec_bytes = off;
  out.rec.assign((size_t)ncomp * off, 0);
  for (int c = 0; c < ncomp; ++c) {
    unsigned char *r = out.rec.data() + (size_t)c * off;
    for (int b = 0; b < m; ++b) {
      const PassHostLayer &H = out.layers[b];
      const size_t g0 = (size_t)c * H.NG;
      for (int q = 0; q < H.NG; ++q) {
        const uint16_t kg = (uint16_t)(H.k[g0 + q] | (H.g[g0 + q] << 8));
        std::memcpy(r + H.off_kg + 2 * q, &kg, 2);
      }
      std::memcpy(r + H.off_src, H.src.data() + g0 * 32, (size_t)H.NG * 64);
      std::memcpy(r + H.off_bias, H.bias.data() + g0 * 32, (size_t)H.NG * 128);
      if (H.off_orow >= 0) std::memcpy(r + H.off_orow, H.orow.data() + g0 * 32, (size_t)H.NG * 128);
    }
  }
}

std::vector<Step> plan_passes(const std::vector<const PackedLayer *> &layers, int32_t n, int cap,
                              int max_m, int tile_floats, int threads,
                              std::vector<PassHost> *built) {
  std::vector<Step> steps = plan_steps(layers, n, cap, max_m);
  std::vector<PassHost> ph(steps.size());
  std::vector<char> done(steps.size(), 0);
  for (;;) {
    std::vector<int> todo;
    for (int i = 0; i < (int)steps.size(); ++i)
      if (steps[i].m > 1 && !done[i]) todo.push_back(i);
    if (todo.empty()) break;
    std::atomic<int> next{0};
    std::vector<std::thread> th;
    const int nt = std::max(1, std::min<int>(threads, (int)todo.size()));
    for (int t = 0; t < nt; ++t)
      th.emplace_back([&] {
        for (int q = next++; q < (int)todo.size(); q = next++)
          build_pass(layers, n, steps[todo[q]], tile_floats, ph[todo[q]]);
      });
    for (auto &x : th) x.join();
    // split passes whose record does not fit (any sub-range of a pass is a pass)
    std::vector<Step> s2;
    std::vector<PassHost> p2;
    std::vector<char> d2;
    for (int i = 0; i < (int)steps.size(); ++i) {
      const Step &S = steps[i];
      if (S.m > 1 && ph[i].rec_bytes > kPassRecMax) {
        Step lo = S, hi = S;
        lo.m = S.m / 2;
        hi.a = S.a + lo.m;
        hi.m = S.m - lo.m;
        for (const Step &x : {lo, hi}) {
          s2.push_back(x);
          p2.emplace_back();
          d2.push_back(x.m == 1);
        }
      } else {
        s2.push_back(S);
        p2.push_back(std::move(ph[i]));
        d2.push_back(1);                    // built in this round or before
      }
    }
    steps.swap(s2);
    ph.swap(p2);
    done.swap(d2);
  }
  if (built) built->swap(ph);
  return steps;
}

}  // namespace sdnn
