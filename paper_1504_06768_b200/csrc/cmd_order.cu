// The reference's 'cmd' ordering: a weighted maximum
// bipartite matching for a zero-free diagonal (ordering.weighted_mbm,
// pkg/src/rhosolve/ordering.py:121-218) followed by an exact greedy column
// minimum-degree ordering on the column-intersection graph
// (ordering.col_min_degree, ordering.py:221-282), used by steady._prepare
// (steady.py:95-107).
//
// Host-native code.  Both algorithms are greedy and strictly sequential --
// every matching / elimination decision depends on all previous ones -- so
// they run on the host, once per structure, like the reference; the
// factorization they order runs on the GPU (rs_factorize).  The results are
// the reference's permutations exactly: the same visiting orders, the same
// tie rules, and |z| = hypot(re, im) as numpy's complex abs computes it.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <deque>
#include <queue>
#include <utility>
#include <vector>

#include "common.cuh"

namespace rs {

namespace {

// (descending magnitude, ascending index) -- numpy lexsort((idx, -mag)) with
// NaN magnitudes last
struct MagIdx {
  double mag;
  int64_t idx;
};
inline bool mag_before(const MagIdx& a, const MagIdx& b) {
  const bool na = std::isnan(a.mag), nb = std::isnan(b.mag);
  if (na != nb) return nb;
  if (!na && a.mag != b.mag) return a.mag > b.mag;
  return a.idx < b.idx;
}

}  // namespace

// Returns 0, or 1 when the matrix is structurally singular.
int weighted_mbm_host(int64_t n, const int64_t* rp, const int64_t* ci, const double2* v,
                      int64_t* forward) {
  // rows of each column (CSC by a stable counting sort: ascending rows)
  std::vector<int64_t> cp(n + 1, 0);
  for (int64_t p = 0; p < rp[n]; ++p) ++cp[ci[p] + 1];
  for (int64_t j = 0; j < n; ++j) cp[j + 1] += cp[j];
  std::vector<MagIdx> colent(rp[n]);
  {
    std::vector<int64_t> fill(cp.begin(), cp.end() - 1);
    for (int64_t i = 0; i < n; ++i)
      for (int64_t p = rp[i]; p < rp[i + 1]; ++p)
        colent[fill[ci[p]]++] = MagIdx{std::hypot(v[p].x, v[p].y), i};
  }
  std::vector<double> col_best(n, 0.0);
  for (int64_t j = 0; j < n; ++j) {
    double best = 0.0;  // max(initial=0.0)
    for (int64_t p = cp[j]; p < cp[j + 1]; ++p)
      if (colent[p].mag > best || std::isnan(colent[p].mag)) best = colent[p].mag;
    col_best[j] = best;
    std::stable_sort(colent.begin() + cp[j], colent.begin() + cp[j + 1], mag_before);
  }
  std::vector<MagIdx> rowent(rp[n]);
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p)
      rowent[p] = MagIdx{std::hypot(v[p].x, v[p].y), ci[p]};
    std::stable_sort(rowent.begin() + rp[i], rowent.begin() + rp[i + 1], mag_before);
  }
  std::vector<int64_t> match_row(n, -1), match_col(n, -1);
  std::vector<char> visited(n, 0);
  // BFS starts: columns by descending best magnitude, ties ascending
  std::vector<MagIdx> starts(n);
  for (int64_t j = 0; j < n; ++j) starts[j] = MagIdx{col_best[j], j};
  std::stable_sort(starts.begin(), starts.end(), mag_before);
  int64_t si = 0, done = 0;
  std::deque<int64_t> q;
  while (done < n) {
    while (si < n && visited[starts[si].idx]) ++si;
    if (si == n) break;
    visited[starts[si].idx] = 1;
    q.push_back(starts[si].idx);
    ++done;
    while (!q.empty()) {
      const int64_t j = q.front();
      q.pop_front();
      for (int64_t p = cp[j]; p < cp[j + 1]; ++p) {
        const int64_t r = colent[p].idx;
        if (match_col[j] < 0 && match_row[r] < 0) {
          match_row[r] = j;
          match_col[j] = r;
        }
        for (int64_t t = rp[r]; t < rp[r + 1]; ++t) {
          const int64_t c2 = rowent[t].idx;
          if (!visited[c2]) {
            visited[c2] = 1;
            q.push_back(c2);
            ++done;
          }
        }
      }
    }
  }
  // complete the matching with BFS augmenting paths over alternating edges
  std::vector<int64_t> reached_from(n);
  std::vector<char> in_tree(n);
  for (int64_t j0 = 0; j0 < n; ++j0) {
    if (match_col[j0] >= 0) continue;
    std::fill(reached_from.begin(), reached_from.end(), -1);
    std::fill(in_tree.begin(), in_tree.end(), 0);
    in_tree[j0] = 1;
    q.clear();
    q.push_back(j0);
    bool augmented = false;
    while (!q.empty() && !augmented) {
      const int64_t j = q.front();
      q.pop_front();
      for (int64_t p = cp[j]; p < cp[j + 1]; ++p) {
        const int64_t r = colent[p].idx;
        if (reached_from[r] >= 0) continue;
        reached_from[r] = j;
        const int64_t jm = match_row[r];
        if (jm < 0) {  // free row: flip the alternating path back to j0
          int64_t rr = r;
          while (true) {
            const int64_t jj = reached_from[rr];
            const int64_t prev = match_col[jj];
            match_row[rr] = jj;
            match_col[jj] = rr;
            if (prev < 0) break;
            rr = prev;
          }
          augmented = true;
          break;
        }
        if (!in_tree[jm]) {
          in_tree[jm] = 1;
          q.push_back(jm);
        }
      }
    }
    if (!augmented) return 1;
  }
  for (int64_t i = 0; i < n; ++i) forward[i] = match_row[i];
  return 0;
}

// Exact greedy minimum degree on the quotient graph: elements start as the
// rows; eliminating column j merges every element touching it into one new
// element (its neighbours); degrees are recomputed exactly for the
// neighbours; ties go to the lowest column.  order[k] = k-th eliminated
// column.
void col_min_degree_host(int64_t n, const int64_t* rp, const int64_t* ci, int64_t* order) {
  std::vector<std::vector<int64_t>> cols_of;  // element -> columns
  std::vector<char> alive;
  cols_of.reserve(2 * n);
  std::vector<std::vector<int64_t>> elems(n);  // column -> elements
  std::vector<int64_t> mark(n, -1);
  int64_t stamp = 0;
  for (int64_t i = 0; i < n; ++i) {
    // a row's distinct columns (CSR rows hold no duplicates)
    std::vector<int64_t> cs(ci + rp[i], ci + rp[i + 1]);
    cols_of.push_back(std::move(cs));
    alive.push_back(rp[i + 1] > rp[i]);
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p) elems[ci[p]].push_back(i);
  }
  auto degree = [&](int64_t j) {
    ++stamp;
    int64_t d = 0;
    mark[j] = stamp;
    for (const int64_t e : elems[j])
      for (const int64_t c : cols_of[e])
        if (mark[c] != stamp) {
          mark[c] = stamp;
          ++d;
        }
    return d;
  };
  std::vector<int64_t> cur(n);
  using Item = std::pair<int64_t, int64_t>;
  std::priority_queue<Item, std::vector<Item>, std::greater<Item>> heap;
  for (int64_t j = 0; j < n; ++j) {
    cur[j] = degree(j);
    heap.push({cur[j], j});
  }
  std::vector<char> eliminated(n, 0);
  std::vector<int64_t> nb;
  for (int64_t k = 0; k < n; ++k) {
    int64_t j;
    while (true) {
      const Item it = heap.top();
      heap.pop();
      j = it.second;
      if (!eliminated[j] && it.first == cur[j]) break;
    }
    order[k] = j;
    eliminated[j] = 1;
    ++stamp;
    mark[j] = stamp;
    nb.clear();
    for (const int64_t e : elems[j])
      for (const int64_t c : cols_of[e])
        if (mark[c] != stamp) {
          mark[c] = stamp;
          nb.push_back(c);
        }
    for (const int64_t e : elems[j]) {
      for (const int64_t c : cols_of[e]) {
        if (c == j) continue;
        auto& ec = elems[c];
        for (size_t t = 0; t < ec.size(); ++t)
          if (ec[t] == e) {
            ec[t] = ec.back();
            ec.pop_back();
            break;
          }
      }
      cols_of[e].clear();
      cols_of[e].shrink_to_fit();
      alive[e] = 0;
    }
    elems[j].clear();
    if (!nb.empty()) {
      const int64_t eid = (int64_t)cols_of.size();
      cols_of.push_back(nb);
      alive.push_back(1);
      for (const int64_t c : nb) elems[c].push_back(eid);
      for (const int64_t c : nb) {
        cur[c] = degree(c);
        heap.push({cur[c], c});
      }
    }
  }
}

}  // namespace rs
