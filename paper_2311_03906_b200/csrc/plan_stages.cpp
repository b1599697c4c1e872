// Host-side planner stages (see plan_stages.hpp).
#include "plan_stages.hpp"

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

namespace symphase::plan {

ChainXf chain_transform(uint64_t n_meas, const std::vector<uint64_t>& row_ptr,
                        const std::vector<uint32_t>& sym_idx, const std::vector<uint64_t>& col_ptr,
                        const std::vector<uint32_t>& col_rows, bool enable) {
  ChainXf x;
  x.parent.assign(n_meas, -1);
  x.depth.assign(n_meas, 0);
  x.rp.assign(1, 0);
  std::vector<uint32_t> cnt(n_meas, 0), touched;
  for (uint64_t k = 0; k < n_meas; ++k) {
    const uint64_t b = row_ptr[k], e = row_ptr[k + 1];
    int64_t best = -1, best_gain = 0;
    if (enable) {
      for (uint64_t i = b; i < e; ++i) {
        const uint32_t sidx = sym_idx[i];
        for (uint64_t t = col_ptr[sidx]; t < col_ptr[sidx + 1]; ++t) {
          const uint32_t j = col_rows[t];
          if (j >= k) break;  // column lists are ascending
          if (cnt[j]++ == 0) touched.push_back(j);
        }
      }
      for (uint32_t j : touched) {
        // |row_k| - |row_k XOR row_j| = 2 overlap - |row_j|
        const int64_t gain = 2 * static_cast<int64_t>(cnt[j]) -
                             static_cast<int64_t>(row_ptr[j + 1] - row_ptr[j]);
        if (gain > best_gain || (gain == best_gain && gain > 0 && j > best)) {
          best_gain = gain;
          best = j;
        }
        cnt[j] = 0;
      }
      touched.clear();
    }
    if (best >= 0) {
      x.parent[k] = static_cast<int32_t>(best);
      x.depth[k] = x.depth[best] + 1;
      x.n_levels = std::max(x.n_levels, x.depth[k] + 1);
      // sorted symmetric difference of row k and row best
      uint64_t i = b, j = row_ptr[best];
      const uint64_t je = row_ptr[best + 1];
      while (i < e || j < je) {
        if (j >= je || (i < e && sym_idx[i] < sym_idx[j])) x.si.push_back(sym_idx[i++]);
        else if (i >= e || sym_idx[j] < sym_idx[i]) x.si.push_back(sym_idx[j++]);
        else { ++i; ++j; }
      }
    } else {
      x.si.insert(x.si.end(), sym_idx.begin() + b, sym_idx.begin() + e);
    }
    x.rp.push_back(x.si.size());
  }
  return x;
}

DrainPlan plan_drain(const std::vector<int32_t>& parent, const std::vector<uint64_t>& det_ptr,
                     const std::vector<uint32_t>& det_meas) {
  const uint64_t n_meas = parent.size();
  DrainPlan P;
  {
    // Heavy-path decomposition of the parent forest (parents precede
    // children, so one reverse sweep gives subtree sizes).
    std::vector<uint32_t> size(n_meas, 1);
    std::vector<int32_t> heavy(n_meas, -1);
    for (uint64_t k = n_meas; k-- > 0;)
      if (parent[k] >= 0) size[parent[k]] += size[k];
    for (uint64_t k = 0; k < n_meas; ++k) {
      const int32_t pa = parent[k];
      if (pa >= 0 && (heavy[pa] < 0 || size[k] > size[heavy[pa]])) heavy[pa] = static_cast<int32_t>(k);
    }
    std::vector<uint32_t> path_of(n_meas, 0), round_of_path;
    std::vector<std::vector<uint16_t>> paths;
    std::vector<int32_t> heads_par;
    for (uint64_t k = 0; k < n_meas; ++k) {
      const int32_t pa = parent[k];
      if (pa >= 0 && heavy[pa] == static_cast<int32_t>(k)) continue;  // continues its parent's path
      const uint32_t id = static_cast<uint32_t>(paths.size());
      paths.emplace_back();
      heads_par.push_back(pa);
      round_of_path.push_back(pa >= 0 ? round_of_path[path_of[pa]] + 1 : 0);
      for (int64_t r = static_cast<int64_t>(k); r >= 0; r = heavy[r]) {
        paths[id].push_back(static_cast<uint16_t>(r));
        path_of[r] = id;
      }
    }
    uint32_t n_rounds = 1;
    for (uint32_t r : round_of_path) n_rounds = std::max(n_rounds, r + 1);
    std::vector<uint32_t> order(paths.size());
    for (uint32_t i = 0; i < order.size(); ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(),
                     [&](uint32_t a, uint32_t b) { return round_of_path[a] < round_of_path[b]; });
    std::vector<uint8_t> keep(n_meas, 0);
    for (uint64_t k = 0; k < n_meas; ++k) {
      const int32_t pa = parent[k];
      if (pa >= 0 && heavy[pa] != static_cast<int32_t>(k)) keep[pa] = 1;  // light child
    }
    // Detectors: {k, parent(k)} (or {k} for a root row) is counted from row
    // k's D value during the rebuild; the others are "general".
    const uint64_t n_det = det_ptr.empty() ? 0 : det_ptr.size() - 1;
    std::vector<uint32_t> det_of_row(n_meas, 0);  // detector index + 1
    std::vector<uint32_t> gdet_ptr{0}, gdet_id;
    std::vector<uint16_t> gdet_rows;
    const bool flat = paths.size() == n_meas && std::all_of(keep.begin(), keep.end(), [](uint8_t v) { return !v; });
    for (uint64_t j = 0; j < n_det; ++j) {
      std::vector<uint32_t> m(det_meas.begin() + det_ptr[j], det_meas.begin() + det_ptr[j + 1]);
      std::sort(m.begin(), m.end());
      std::vector<uint32_t> odd;  // a measurement listed twice cancels
      for (size_t i = 0; i < m.size();) {
        size_t e = i;
        while (e < m.size() && m[e] == m[i]) ++e;
        if ((e - i) & 1) odd.push_back(m[i]);
        i = e;
      }
      int64_t row = -1;
      if (!flat && n_det < 0x7FFF) {
        if (odd.size() == 1 && parent[odd[0]] < 0) row = odd[0];
        if (odd.size() == 2 && parent[odd[1]] == static_cast<int32_t>(odd[0])) row = odd[1];
        if (row >= 0 && det_of_row[row]) row = -1;  // the row already counts another detector
      }
      if (row >= 0) {
        det_of_row[row] = static_cast<uint32_t>(j + 1);
      } else {
        for (uint32_t r : odd) gdet_rows.push_back(static_cast<uint16_t>(r));
        gdet_ptr.push_back(static_cast<uint32_t>(gdet_rows.size()));
        gdet_id.push_back(static_cast<uint32_t>(j));
      }
    }
    // the legacy drain clears rows as it goes: keep the general detectors'
    // rows until the tile ends
    if (!flat)
      for (uint16_t r : gdet_rows) keep[r] = 1;
    std::vector<uint32_t> path_rows;
    std::vector<uint32_t> path_ptr{0}, round_ptr(n_rounds + 1, 0);
    std::vector<uint16_t> keep_rows;
    std::vector<int32_t> path_par;
    for (uint32_t id : order) {
      for (uint16_t r : paths[id]) {
        path_rows.push_back(r | (det_of_row[r] << 16) | (keep[r] ? 0x80000000u : 0u));
        if (keep[r]) keep_rows.push_back(r);
      }
      path_ptr.push_back(static_cast<uint32_t>(path_rows.size()));
      path_par.push_back(heads_par[id]);
      round_ptr[round_of_path[id] + 1]++;
    }
    for (uint32_t r = 0; r < n_rounds; ++r) round_ptr[r + 1] += round_ptr[r];
    for (int i = 0; i < 4; ++i) path_rows.push_back(0);  // prefetch padding: walks read past a path
    P.n_paths = static_cast<uint32_t>(paths.size());
    P.n_rounds = n_rounds;
    P.flat = paths.size() == n_meas && keep_rows.empty();
    P.n_det = static_cast<uint32_t>(n_det);
    P.path_rows = std::move(path_rows);
    P.path_ptr = std::move(path_ptr);
    P.round_ptr = std::move(round_ptr);
    P.path_par = std::move(path_par);
    P.keep_rows = std::move(keep_rows);
    P.gdet_ptr = std::move(gdet_ptr);
    P.gdet_id = std::move(gdet_id);
    P.gdet_rows = std::move(gdet_rows);
  }
  return P;
}

double mechanism_rate(uint8_t dist, double p) {
  double q = -1.0;
  if (dist == 3 && p > 0.0 && p < 0.75) q = 0.5 * (1.0 - std::sqrt(1.0 - 4.0 * p / 3.0));
  if (dist == 4 && p > 0.0 && p < 15.0 / 16.0) q = 0.5 * (1.0 - std::pow(1.0 - 16.0 * p / 15.0, 0.125));
  return q > 0.0 && q < 0.5 ? q : -1.0;
}

}  // namespace symphase::plan
