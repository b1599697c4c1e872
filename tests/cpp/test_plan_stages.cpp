// CPU unit tests of the planner's host stages (paper_2311_03906_b200/csrc/
// plan_stages.cpp): the chain transform M = L·D, the drain plan (heavy paths
// + detector classification) and the exact DEPOLARIZE mechanism rates.
// Prints one line per failed check; exits non-zero on any failure.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <random>
#include <set>
#include <vector>

#include "plan_stages.hpp"

using namespace symphase::plan;

static int g_fail = 0, g_checks = 0;
#define CHECK(x)                                                    \
  do {                                                              \
    ++g_checks;                                                     \
    if (!(x)) {                                                     \
      ++g_fail;                                                     \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #x);      \
    }                                                               \
  } while (0)

struct Csr {
  std::vector<uint64_t> rp{0};
  std::vector<uint32_t> si;
  std::vector<uint64_t> cp;
  std::vector<uint32_t> cr;
};

// Random rows, with "rounds": row k often repeats an earlier row plus a few
// symbols (the structure the chain transform is for).
static Csr random_rows(std::mt19937_64& rng, uint32_t n, uint32_t v) {
  Csr c;
  std::vector<std::vector<uint32_t>> rows;
  for (uint32_t k = 0; k < n; ++k) {
    std::set<uint32_t> r;
    if (k && rng() % 3) {
      const auto& base = rows[rng() % k];
      r.insert(base.begin(), base.end());
    }
    for (int t = 0, m = 1 + rng() % 6; t < m; ++t) {
      const uint32_t s = rng() % v;
      if (!r.erase(s)) r.insert(s);
    }
    rows.emplace_back(r.begin(), r.end());
    c.si.insert(c.si.end(), r.begin(), r.end());
    c.rp.push_back(c.si.size());
  }
  c.cp.assign(v + 1, 0);
  for (uint32_t s : c.si) c.cp[s + 1]++;
  for (uint32_t i = 0; i < v; ++i) c.cp[i + 1] += c.cp[i];
  c.cr.resize(c.si.size());
  std::vector<uint64_t> fill(c.cp.begin(), c.cp.end() - 1);
  for (uint32_t k = 0; k < n; ++k)
    for (uint64_t i = c.rp[k]; i < c.rp[k + 1]; ++i) c.cr[fill[c.si[i]]++] = k;
  return c;
}

static std::vector<uint32_t> row_of(const std::vector<uint64_t>& rp, const std::vector<uint32_t>& si,
                                    uint32_t k) {
  return {si.begin() + rp[k], si.begin() + rp[k + 1]};
}

static std::vector<uint32_t> symdiff(const std::vector<uint32_t>& a, const std::vector<uint32_t>& b) {
  std::vector<uint32_t> o;
  std::set_symmetric_difference(a.begin(), a.end(), b.begin(), b.end(), std::back_inserter(o));
  return o;
}

static void test_chain(std::mt19937_64& rng) {
  for (int trial = 0; trial < 30; ++trial) {
    const uint32_t n = 1 + rng() % 300, v = 1 + rng() % 200;
    Csr c = random_rows(rng, n, v);
    ChainXf X = chain_transform(n, c.rp, c.si, c.cp, c.cr, true);
    CHECK(X.parent.size() == n && X.rp.size() == n + 1);
    for (uint32_t k = 0; k < n; ++k) {
      const auto m = row_of(c.rp, c.si, k), d = row_of(X.rp, X.si, k);
      CHECK(std::is_sorted(d.begin(), d.end()));
      if (X.parent[k] >= 0) {
        CHECK(X.parent[k] < static_cast<int32_t>(k));
        CHECK(d == symdiff(m, row_of(c.rp, c.si, X.parent[k])));
        CHECK(d.size() < m.size());
      } else {
        CHECK(d == m);
      }
      // out[k] = d[k] ^ out[p(k)] rebuilds row k
      std::vector<uint32_t> acc = d;
      for (int32_t p = X.parent[k]; p >= 0; p = X.parent[p]) acc = symdiff(acc, row_of(X.rp, X.si, p));
      CHECK(acc == m);
    }
    ChainXf Y = chain_transform(n, c.rp, c.si, c.cp, c.cr, false);
    CHECK(Y.si == c.si && std::all_of(Y.parent.begin(), Y.parent.end(), [](int32_t p) { return p < 0; }));
  }
}

// The measurements a detector XORs: those listed an odd number of times.
static std::vector<uint32_t> odd_members(std::vector<uint32_t> d) {
  std::sort(d.begin(), d.end());
  std::vector<uint32_t> odd;
  for (size_t i = 0; i < d.size();) {
    size_t e = i;
    while (e < d.size() && d[e] == d[i]) ++e;
    if ((e - i) & 1) odd.push_back(d[i]);
    i = e;
  }
  return odd;
}

static void test_drain(std::mt19937_64& rng) {
  for (int trial = 0; trial < 60; ++trial) {
    const uint32_t n = 1 + rng() % 400;
    std::vector<int32_t> parent(n, -1);
    const bool flat_forest = trial % 10 == 0;
    for (uint32_t k = 1; k < n && !flat_forest; ++k)
      if (rng() % 4) parent[k] = static_cast<int32_t>(k > 30 && rng() % 2 ? k - 1 - rng() % 30 : rng() % k);
    // detectors: row-shaped {k, p(k)}, roots {k}, and general ones
    std::vector<uint64_t> dptr{0};
    std::vector<uint32_t> dm;
    std::vector<std::vector<uint32_t>> dets;
    for (int j = 0, nd = rng() % 60; j < nd; ++j) {
      std::vector<uint32_t> d;
      const uint32_t k = rng() % n;
      switch (rng() % 4) {
        case 0: if (parent[k] >= 0) d = {static_cast<uint32_t>(parent[k]), k}; else d = {k}; break;
        case 1: d = {k, k, static_cast<uint32_t>(rng() % n)}; break;  // a repeat cancels
        default: for (int t = 0, m = rng() % 5; t < m; ++t) d.push_back(rng() % n);
      }
      dets.push_back(d);
      dm.insert(dm.end(), d.begin(), d.end());
      dptr.push_back(dm.size());
    }
    DrainPlan P = plan_drain(parent, dptr, dm);
    CHECK(P.path_ptr.size() == P.n_paths + 1 && P.path_par.size() == P.n_paths);
    CHECK(P.path_rows.size() == static_cast<size_t>(n) + 4);
    CHECK(P.round_ptr.size() == P.n_rounds + 1 && P.round_ptr.front() == 0 && P.round_ptr.back() == P.n_paths);
    std::vector<int> seen(n, 0), round_of_row(n, -1), det_row(n, 0);
    std::vector<uint8_t> kept(n, 0);
    for (uint32_t r = 0; r < P.n_rounds; ++r)
      for (uint32_t p = P.round_ptr[r]; p < P.round_ptr[r + 1]; ++p) {
        const int32_t head_par = P.path_par[p];
        CHECK(head_par < 0 || (round_of_row[head_par] >= 0 && round_of_row[head_par] < static_cast<int>(r)));
        int32_t prev = head_par;
        for (uint32_t x = P.path_ptr[p]; x < P.path_ptr[p + 1]; ++x) {
          const uint32_t e = P.path_rows[x], k = e & 0xFFFFu;
          CHECK(k < n);
          if (k >= n) continue;
          ++seen[k];
          CHECK(parent[k] == prev);  // a path is a parent chain
          prev = static_cast<int32_t>(k);
          round_of_row[k] = static_cast<int>(r);
          det_row[k] = (e >> 16) & 0x7FFF;
          kept[k] = e >> 31;
        }
      }
    for (uint32_t k = 0; k < n; ++k) CHECK(seen[k] == 1);
    std::set<uint16_t> keep_set(P.keep_rows.begin(), P.keep_rows.end());
    for (uint32_t k = 0; k < n; ++k) CHECK((kept[k] != 0) == (keep_set.count(k) != 0));
    bool any_parent = std::any_of(parent.begin(), parent.end(), [](int32_t p) { return p >= 0; });
    CHECK(P.flat == !any_parent);
    // detector classification: every detector is a row detector or general,
    // exactly once, and each is counted from the right rows
    CHECK(P.n_det == dets.size());
    std::vector<int> counted(dets.size(), 0);
    for (uint32_t k = 0; k < n; ++k)
      if (det_row[k]) {
        const uint32_t j = det_row[k] - 1;
        ++counted[j];
        std::vector<uint32_t> d = odd_members(dets[j]);
        std::vector<uint32_t> want = parent[k] >= 0 ? std::vector<uint32_t>{static_cast<uint32_t>(parent[k]), k}
                                                    : std::vector<uint32_t>{k};
        CHECK(d == want);
      }
    for (size_t g = 0; g < P.gdet_id.size(); ++g) {
      const uint32_t j = P.gdet_id[g];
      ++counted[j];
      const std::vector<uint32_t> odd = odd_members(dets[j]);
      std::vector<uint32_t> rows(P.gdet_rows.begin() + P.gdet_ptr[g], P.gdet_rows.begin() + P.gdet_ptr[g + 1]);
      CHECK(rows == odd);
      if (!P.flat)
        for (uint32_t r : rows) CHECK(kept[r]);  // the legacy drain must keep them
    }
    for (size_t j = 0; j < dets.size(); ++j) CHECK(counted[j] == 1);
  }
}

// P(XOR of independently fired mechanisms = v) for the n = 2^b - 1 patterns.
static void test_mechanisms() {
  for (int dist : {3, 4}) {
    const int bits = dist == 3 ? 2 : 4, npat = (1 << bits) - 1;
    for (double p : {1e-6, 1e-3, 0.01, 0.1, 0.3, 0.5, dist == 3 ? 0.7 : 0.9}) {
      const double q = mechanism_rate(static_cast<uint8_t>(dist), p);
      CHECK(q > 0.0 && q < 0.5);
      std::vector<double> pv(1 << bits, 0.0);
      for (uint32_t subset = 0; subset < (1u << npat); ++subset) {
        double pr = 1.0;
        uint32_t v = 0;
        for (int m = 0; m < npat; ++m) {
          const bool on = (subset >> m) & 1u;
          pr *= on ? q : 1.0 - q;
          if (on) v ^= static_cast<uint32_t>(m + 1);
        }
        pv[v] += pr;
      }
      CHECK(std::fabs(pv[0] - (1.0 - p)) < 1e-12);
      for (int v = 1; v <= npat; ++v) CHECK(std::fabs(pv[v] - p / npat) < 1e-12);
    }
    CHECK(mechanism_rate(static_cast<uint8_t>(dist), 0.0) < 0);
    CHECK(mechanism_rate(static_cast<uint8_t>(dist), dist == 3 ? 0.75 : 15.0 / 16.0) < 0);
  }
  CHECK(mechanism_rate(1, 0.1) < 0);  // Bernoulli: nothing to decompose
}

int main() {
  std::mt19937_64 rng(2311);
  test_chain(rng);
  test_drain(rng);
  test_mechanisms();
  std::printf("%d checks, %d failed\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
