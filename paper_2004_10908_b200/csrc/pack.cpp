// pack.cpp -- create-time validation and packing of one weight layer W_l
// (dataset part "1920 layers of neurons stored in sparse
// matrices").  Not in the timed region.
//
// Output layout: columns with identical ascending
// source lists are merged into groups of <= 32 (the RadiX-Net-shaped layers are
// N/32 dense 32x32 blocks), so a warp loads a group's source rows once and
// produces all of its member columns.  Each member's chain still runs over its
// own sources in ascending k, so the arithmetic is the canonical one.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>

#include "../../include/sdnn.h"
#include "sdnn_internal.h"

namespace sdnn {
namespace {

inline uint32_t fbits(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  return u;
}

uint64_t hash_list(const int32_t *s, int32_t len) {
  uint64_t h = 1469598103934665603ull ^ (uint64_t)len;
  for (int32_t i = 0; i < len; ++i) {
    h ^= (uint64_t)(uint32_t)s[i];
    h *= 1099511628211ull;
    h ^= h >> 29;
  }
  return h;
}

}  // namespace

int pack_layer(int32_t n, const LayerIn &in, const float *bias, bool allow_groups,
               PackedLayer &out, std::string &msg) {
  out = PackedLayer();
  out.n = n;
  // ---- 1. column lists (ascending source k) -------------------------------
  std::vector<int64_t> cptr(n + 1, 0);
  std::vector<int32_t> csrc;
  std::vector<float> cval;
  const bool has_val = in.val != nullptr;
  if (!has_val && !std::isfinite(in.uniform_value)) {
    msg = "uniform_value is not finite";
    return SDNN_E_FORMAT;
  }
  if (in.format == SDNN_W_CSR) {
    if (!in.rowptr || (!in.idx && in.rowptr[n] > 0)) {
      msg = "CSR layer needs rowptr and idx";
      return SDNN_E_ARG;
    }
    if (in.rowptr[0] != 0) {
      msg = "rowptr[0] != 0";
      return SDNN_E_FORMAT;
    }
    for (int32_t k = 0; k < n; ++k)
      if (in.rowptr[k + 1] < in.rowptr[k]) {
        msg = "rowptr not non-decreasing at row " + std::to_string(k);
        return SDNN_E_FORMAT;
      }
    const int64_t nnz = in.rowptr[n];
    for (int64_t e = 0; e < nnz; ++e) {
      const int32_t j = in.idx[e];
      if (j < 0 || j >= n) {
        msg = "column index out of range at entry " + std::to_string(e);
        return SDNN_E_FORMAT;
      }
      if (has_val && !std::isfinite(in.val[e])) {
        msg = "non-finite weight at entry " + std::to_string(e);
        return SDNN_E_FORMAT;
      }
      cptr[j + 1]++;
    }
    for (int32_t j = 0; j < n; ++j) cptr[j + 1] += cptr[j];
    csrc.resize(nnz);
    if (has_val) cval.resize(nnz);
    std::vector<int64_t> fill(cptr.begin(), cptr.end() - 1);
    for (int32_t k = 0; k < n; ++k)            // rows in ascending k => stable
      for (int64_t e = in.rowptr[k]; e < in.rowptr[k + 1]; ++e) {
        const int64_t p = fill[in.idx[e]]++;
        csrc[p] = k;
        if (has_val) cval[p] = in.val[e];
      }
  } else if (in.format == SDNN_W_ELLCOL) {
    if (in.ell_k < 0) {
      msg = "ell_k < 0";
      return SDNN_E_ARG;
    }
    if (in.ell_k > 0 && !in.idx) {
      msg = "ELLCOL layer needs idx";
      return SDNN_E_ARG;
    }
    const int32_t ek = in.ell_k;
    std::vector<std::pair<int32_t, float>> tmp(ek);
    csrc.reserve((size_t)n * ek);
    if (has_val) cval.reserve((size_t)n * ek);
    for (int32_t j = 0; j < n; ++j) {
      int32_t c = 0;
      for (int32_t t = 0; t < ek; ++t) {
        const int32_t k = in.idx[(int64_t)j * ek + t];
        if (k == -1) continue;
        if (k < 0 || k >= n) {
          msg = "source index out of range in column " + std::to_string(j);
          return SDNN_E_FORMAT;
        }
        const float v = has_val ? in.val[(int64_t)j * ek + t] : 0.f;
        if (has_val && !std::isfinite(v)) {
          msg = "non-finite weight in column " + std::to_string(j);
          return SDNN_E_FORMAT;
        }
        tmp[c++] = {k, v};
      }
      std::sort(tmp.begin(), tmp.begin() + c,
                [](const auto &a, const auto &b) { return a.first < b.first; });
      for (int32_t t = 0; t < c; ++t) {
        csrc.push_back(tmp[t].first);
        if (has_val) cval.push_back(tmp[t].second);
      }
      cptr[j + 1] = cptr[j] + c;
    }
  } else {
    msg = "unknown layer format";
    return SDNN_E_ARG;
  }
  const int64_t nnz = cptr[n];
  out.nnz = nnz;
  // duplicates: a repeated (k, j) is adjacent in column j's ascending list
  for (int32_t j = 0; j < n; ++j)
    for (int64_t p = cptr[j] + 1; p < cptr[j + 1]; ++p)
      if (csrc[p] == csrc[p - 1]) {
        msg = "duplicate entry (k=" + std::to_string(csrc[p]) + ", j=" + std::to_string(j) + ")";
        return SDNN_E_FORMAT;
      }
  // ---- 2. uniform value detection (bit-identical) --------------------------
  if (!has_val) {
    out.uniform = true;
    out.wu = in.uniform_value;
  } else if (nnz == 0) {
    out.uniform = true;
    out.wu = 0.f;
  } else {
    const uint32_t b0 = fbits(cval[0]);
    out.uniform = true;
    for (int64_t p = 1; p < nnz && out.uniform; ++p) out.uniform = fbits(cval[p]) == b0;
    out.wu = cval[0];
  }
  // ---- 3. bias ---------------------------------------------------------------
  out.bias.assign(bias, bias + n);
  for (int32_t j = 0; j < n; ++j) {
    if (!std::isfinite(bias[j])) {
      msg = "non-finite bias at neuron " + std::to_string(j);
      return SDNN_E_FORMAT;
    }
    if (bias[j] > 0.f) out.bias_nonpos = false;
  }
  // ---- 4. groups of columns with identical source lists ---------------------
  std::vector<std::vector<int32_t>> groups;
  if (allow_groups) {
    std::vector<uint64_t> h(n);
    for (int32_t j = 0; j < n; ++j)
      h[j] = hash_list(csrc.data() + cptr[j], (int32_t)(cptr[j + 1] - cptr[j]));
    std::vector<int32_t> order(n);
    std::iota(order.begin(), order.end(), 0);
    std::sort(order.begin(), order.end(), [&](int32_t a, int32_t b) {
      return h[a] != h[b] ? h[a] < h[b] : a < b;
    });
    auto same = [&](int32_t a, int32_t b) {
      const int64_t la = cptr[a + 1] - cptr[a], lb = cptr[b + 1] - cptr[b];
      return la == lb && std::equal(csrc.begin() + cptr[a], csrc.begin() + cptr[a + 1],
                                    csrc.begin() + cptr[b]);
    };
    for (int32_t s = 0; s < n;) {
      int32_t e = s;
      while (e < n && h[order[e]] == h[order[s]]) ++e;
      // exact classes inside a hash run (collisions are split apart)
      std::vector<std::vector<int32_t>> cls;
      for (int32_t q = s; q < e; ++q) {
        const int32_t j = order[q];
        bool placed = false;
        for (auto &c : cls)
          if (same(c[0], j)) {
            c.push_back(j);
            placed = true;
            break;
          }
        if (!placed) cls.push_back({j});
      }
      for (auto &c : cls)                      // members ascending (order is by j)
        for (size_t o = 0; o < c.size(); o += kMaxGroup)
          groups.emplace_back(c.begin() + o, c.begin() + std::min(c.size(), o + kMaxGroup));
      s = e;
    }
    std::sort(groups.begin(), groups.end(),
              [](const auto &a, const auto &b) { return a[0] < b[0]; });
  } else {
    groups.resize(n);
    for (int32_t j = 0; j < n; ++j) groups[j] = {j};
  }
  // ---- 5. flatten --------------------------------------------------------------
  const int32_t G = (int32_t)groups.size();
  out.ngroups = G;
  int32_t kmax = 0, gmax = 0;
  for (auto &g : groups) {
    kmax = std::max<int32_t>(kmax, (int32_t)(cptr[g[0] + 1] - cptr[g[0]]));
    gmax = std::max<int32_t>(gmax, (int32_t)g.size());
  }
  out.kmax = kmax;
  out.gmax = gmax;
  out.src.assign((size_t)G * std::max(kmax, 1), 0);
  out.col.assign((size_t)G * std::max(gmax, 1), -1);
  out.gk.resize(G);
  out.gg.resize(G);
  if (!out.uniform) out.val.assign((size_t)G * std::max(gmax, 1) * std::max(kmax, 1), 0.f);
  out.regular = true;
  for (int32_t g = 0; g < G; ++g) {
    const auto &m = groups[g];
    const int32_t j0 = m[0];
    const int32_t kg = (int32_t)(cptr[j0 + 1] - cptr[j0]);
    out.gk[g] = kg;
    out.gg[g] = (int32_t)m.size();
    if (kg != kmax || (int32_t)m.size() != gmax) out.regular = false;
    for (int32_t t = 0; t < kg; ++t) out.src[(size_t)g * kmax + t] = (uint16_t)csrc[cptr[j0] + t];
    for (size_t q = 0; q < m.size(); ++q) {
      out.col[(size_t)g * gmax + q] = m[q];
      if (!out.uniform)
        for (int32_t t = 0; t < kg; ++t)
          out.val[((size_t)g * kmax + t) * gmax + q] = cval[cptr[m[q]] + t];
    }
  }
  // per-group member biases (contiguous per group: staged by TMA next to the
  // weights in k_layer_bulkw)
  if (!out.uniform) {
    out.gbias.assign((size_t)G * std::max(gmax, 1), 0.f);
    for (int32_t g = 0; g < G; ++g)
      for (int32_t q = 0; q < out.gg[g]; ++q) out.gbias[(size_t)g * gmax + q] = bias[out.col[(size_t)g * gmax + q]];
  }
  return SDNN_OK;
}

bool saturation_preserving(const PackedLayer &p, float ymax) {
  for (int32_t g = 0; g < p.ngroups; ++g) {
    const int K = p.gk[g], G = p.gg[g];
    for (int m = 0; m < G; ++m) {
      float acc = 0.f;                           // the canonical chain on all-ymax inputs
      for (int t = 0; t < K; ++t) {
        const float w = p.uniform ? p.wu : p.val[((size_t)g * p.kmax + t) * p.gmax + m];
        acc = std::fmaf(ymax, w, acc);
      }
      const float z = acc + p.bias[p.col[(size_t)g * p.gmax + m]];
      if (!(z >= ymax)) return false;
    }
  }
  // a column outside every group cannot exist (each output belongs to one group)
  return true;
}

}  // namespace sdnn
