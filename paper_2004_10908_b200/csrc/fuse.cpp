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
#include <numeric>

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
        while (a + m < L && m < max_m && fusable(*layers[a + m])) {
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
                int buf_floats, int min_t, PassHost &out) {
  const int m = s.m;
  UF uf;
  uf.init((int64_t)(m + 1) * n);
  for (int b = 0; b < m; ++b) add_layer(uf, *layers[s.a + b], n, b);
  // components that own at least one group (have outputs); dense ids by smallest node
  std::vector<int32_t> comp_of_root((size_t)(m + 1) * n, -1);
  int ncomp = 0;
  for (int b = 0; b < m; ++b) {
    const PackedLayer &p = *layers[s.a + b];
    for (int32_t g = 0; g < p.ngroups; ++g) {
      const int32_t r = uf.find((int32_t)((int64_t)(b + 1) * n + p.col[(size_t)g * p.gmax]));
      if (comp_of_root[r] < 0) comp_of_root[r] = ncomp++;
    }
  }
  // local row index of every node: order by neuron id within (component, boundary)
  std::vector<int32_t> local((size_t)(m + 1) * n, -1);
  std::vector<std::vector<int32_t>> rows_in(ncomp), rows_out(ncomp);
  std::vector<int32_t> fill((size_t)ncomp * (m + 1), 0);
  int R = 0;
  for (int b = 0; b <= m; ++b)
    for (int32_t i = 0; i < n; ++i) {
      const int64_t node = (int64_t)b * n + i;
      const int32_t c = comp_of_root[uf.find((int32_t)node)];
      if (c < 0) continue;                      // input neuron feeding nothing in this pass
      const int32_t li = fill[(size_t)c * (m + 1) + b]++;
      local[node] = li;
      R = std::max(R, li + 1);
      if (b == 0) rows_in[c].push_back(i);
      if (b == m) rows_out[c].push_back(i);
    }
  out = PassHost();
  out.a = s.a;
  out.m = m;
  out.ncomp = ncomp;
  out.R = R;
  int rin = 0, rout = 0;
  for (int c = 0; c < ncomp; ++c) {
    rin = std::max<int>(rin, (int)rows_in[c].size());
    rout = std::max<int>(rout, (int)rows_out[c].size());
  }
  out.rin = std::max(rin, 1);
  out.rout = std::max(rout, 1);
  // positions per item: one smem buffer (buf_floats) per component tile
  int T = 512;
  while (T > min_t && (int64_t)R * T > buf_floats) T >>= 1;
  out.T = T;
  out.in_rows.assign((size_t)ncomp * out.rin, -1);
  out.in_count.assign(ncomp, 0);
  out.out_rows.assign((size_t)ncomp * out.rout, -1);
  for (int c = 0; c < ncomp; ++c) {
    std::copy(rows_in[c].begin(), rows_in[c].end(), out.in_rows.begin() + (size_t)c * out.rin);
    out.in_count[c] = (int32_t)rows_in[c].size();
    std::copy(rows_out[c].begin(), rows_out[c].end(), out.out_rows.begin() + (size_t)c * out.rout);
  }
  out.layers.resize(m);
  for (int b = 0; b < m; ++b) {
    const PackedLayer &p = *layers[s.a + b];
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
    H.dst.assign((size_t)ncomp * NG * 32, 0);
    H.bias.assign((size_t)ncomp * NG * 32, 0.f);
    H.k.assign((size_t)ncomp * NG, 0);
    H.g.assign((size_t)ncomp * NG, 0);
    const int64_t in0 = (int64_t)b * n, out0 = (int64_t)(b + 1) * n;
    for (int c = 0; c < ncomp; ++c)
      for (size_t q = 0; q < groups[c].size(); ++q) {
        const int32_t g = groups[c][q];
        const size_t rec = (size_t)c * NG + q;
        const int K = p.gk[g], G = p.gg[g];
        H.k[rec] = (uint8_t)K;
        H.g[rec] = (uint8_t)G;
        for (int t = 0; t < K; ++t)        // keeps the ascending source order (canonical chain)
          H.src[rec * 32 + t] = (uint16_t)local[in0 + p.src[(size_t)g * p.kmax + t]];
        for (int u = 0; u < G; ++u) {
          const int32_t j = p.col[(size_t)g * p.gmax + u];
          H.dst[rec * 32 + u] = (uint16_t)local[out0 + j];
          H.bias[rec * 32 + u] = p.bias[j];
        }
      }
  }
}

}  // namespace sdnn
