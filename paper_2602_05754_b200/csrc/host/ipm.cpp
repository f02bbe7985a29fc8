#include "ipm.hpp"

#include <algorithm>
#include <cmath>
#include <deque>
#include <limits>
#include <numeric>
#include <stdexcept>
#include <cstdio>
#include <cstdlib>

namespace pipefreeze::ipm {

namespace {

using Vec = std::vector<double>;

// Reverse Cuthill-McKee over the co-occurrence graph of the sparse rows.
std::vector<int> rcm_order(int n, const std::vector<Row>& rows) {
  std::vector<std::vector<int>> adj(static_cast<std::size_t>(n));
  for (const auto& r : rows) {
    if (r.dense) continue;
    for (int a : r.idx)
      for (int b : r.idx)
        if (a != b) adj[static_cast<std::size_t>(a)].push_back(b);
  }
  for (auto& l : adj) {
    std::sort(l.begin(), l.end());
    l.erase(std::unique(l.begin(), l.end()), l.end());
  }
  auto deg = [&](int v) { return static_cast<int>(adj[static_cast<std::size_t>(v)].size()); };
  std::vector<int> order;
  order.reserve(static_cast<std::size_t>(n));
  std::vector<char> seen(static_cast<std::size_t>(n), 0);
  auto bfs = [&](int root, std::vector<int>& out, std::vector<int>& level) {
    out.clear();
    std::vector<char> mark(static_cast<std::size_t>(n), 0);
    std::deque<int> q{root};
    mark[static_cast<std::size_t>(root)] = 1;
    level.assign(static_cast<std::size_t>(n), -1);
    level[static_cast<std::size_t>(root)] = 0;
    while (!q.empty()) {
      const int v = q.front();
      q.pop_front();
      out.push_back(v);
      std::vector<int> nb;
      for (int w : adj[static_cast<std::size_t>(v)])
        if (!mark[static_cast<std::size_t>(w)] && !seen[static_cast<std::size_t>(w)]) {
          mark[static_cast<std::size_t>(w)] = 1;
          nb.push_back(w);
        }
      std::sort(nb.begin(), nb.end(), [&](int a, int b) { return deg(a) != deg(b) ? deg(a) < deg(b) : a < b; });
      for (int w : nb) {
        level[static_cast<std::size_t>(w)] = level[static_cast<std::size_t>(v)] + 1;
        q.push_back(w);
      }
    }
  };
  std::vector<int> comp, level;
  for (int start = 0; start < n; ++start) {
    if (seen[static_cast<std::size_t>(start)]) continue;
    // pseudo-peripheral root: repeat BFS from the deepest, lowest-degree node
    int root = start;
    int depth = -1;
    for (int rep = 0; rep < 4; ++rep) {
      bfs(root, comp, level);
      int far = root, fd = 0;
      for (int v : comp) {
        const int l = level[static_cast<std::size_t>(v)];
        if (l > fd || (l == fd && deg(v) < deg(far))) {
          fd = l;
          far = v;
        }
      }
      if (fd <= depth) break;
      depth = fd;
      root = far;
    }
    bfs(root, comp, level);
    for (int v : comp) seen[static_cast<std::size_t>(v)] = 1;
    order.insert(order.end(), comp.begin(), comp.end());
  }
  std::reverse(order.begin(), order.end());
  return order;  // order[new] = old
}

class Skyline {
 public:
  Skyline(int n, const std::vector<Row>& rows, const std::vector<int>& perm) : n_(n) {
    iperm_.assign(static_cast<std::size_t>(n), 0);
    for (int i = 0; i < n; ++i) iperm_[static_cast<std::size_t>(perm[static_cast<std::size_t>(i)])] = i;
    first_.resize(static_cast<std::size_t>(n));
    std::iota(first_.begin(), first_.end(), 0);
    for (const auto& r : rows) {
      if (r.dense || r.idx.empty()) continue;
      int lo = n;
      for (int v : r.idx) lo = std::min(lo, iperm_[static_cast<std::size_t>(v)]);
      for (int v : r.idx) {
        auto& f = first_[static_cast<std::size_t>(iperm_[static_cast<std::size_t>(v)])];
        f = std::min(f, lo);
      }
    }
    off_.resize(static_cast<std::size_t>(n) + 1);
    off_[0] = 0;
    for (int i = 0; i < n; ++i)
      off_[static_cast<std::size_t>(i) + 1] = off_[static_cast<std::size_t>(i)] + (i - first_[static_cast<std::size_t>(i)] + 1);
    env_.assign(off_[static_cast<std::size_t>(n)], 0.0);
  }

  std::size_t envelope() const { return env_.size(); }

  void clear() { std::fill(env_.begin(), env_.end(), 0.0); }

  // Accumulate d * a a^T for one sparse row.
  void add_row(const Row& r, double d) {
    const std::size_t k = r.idx.size();
    for (std::size_t p = 0; p < k; ++p) {
      const int ip = iperm_[static_cast<std::size_t>(r.idx[p])];
      for (std::size_t q = 0; q < k; ++q) {
        const int iq = iperm_[static_cast<std::size_t>(r.idx[q])];
        if (iq > ip) continue;
        at(ip, iq) += d * r.val[p] * r.val[q];
      }
    }
  }

  void add_diag(int v, double d) { at(iperm_[static_cast<std::size_t>(v)], iperm_[static_cast<std::size_t>(v)]) += d; }

  // In-place L L^T factorisation; tiny pivots are replaced by a huge value so
  // the corresponding solution component vanishes (standard IPM safeguard).
  void factor() {
    for (int i = 0; i < n_; ++i) {
      double* Li = row(i);
      const int fi = first_[static_cast<std::size_t>(i)];
      const double aii = Li[i];
      for (int j = fi; j < i; ++j) {
        const double* Lj = row(j);
        const int k0 = std::max(fi, first_[static_cast<std::size_t>(j)]);
        double s = Li[j];
        for (int k = k0; k < j; ++k) s -= Li[k] * Lj[k];
        Li[j] = s / Lj[j];
      }
      double d = aii;
      for (int k = fi; k < i; ++k) d -= Li[k] * Li[k];
      if (!(d > 1e-30 * std::max(1.0, std::abs(aii)))) d = 1e128;
      Li[i] = std::sqrt(d);
    }
  }

  // Solve (L L^T) x = b in the ORIGINAL variable order.
  void solve(const Vec& b, Vec& x) const {
    Vec y(static_cast<std::size_t>(n_));
    for (int i = 0; i < n_; ++i) y[static_cast<std::size_t>(i)] = b[static_cast<std::size_t>(perm_of(i))];
    for (int i = 0; i < n_; ++i) {
      const double* Li = row(i);
      double s = y[static_cast<std::size_t>(i)];
      for (int k = first_[static_cast<std::size_t>(i)]; k < i; ++k) s -= Li[k] * y[static_cast<std::size_t>(k)];
      y[static_cast<std::size_t>(i)] = s / Li[i];
    }
    for (int i = n_ - 1; i >= 0; --i) {
      const double* Li = row(i);
      const double xi = y[static_cast<std::size_t>(i)] / Li[i];
      y[static_cast<std::size_t>(i)] = xi;
      for (int k = first_[static_cast<std::size_t>(i)]; k < i; ++k) y[static_cast<std::size_t>(k)] -= Li[k] * xi;
    }
    x.assign(static_cast<std::size_t>(n_), 0.0);
    for (int i = 0; i < n_; ++i) x[static_cast<std::size_t>(perm_of(i))] = y[static_cast<std::size_t>(i)];
  }

  void set_perm(const std::vector<int>& perm) { perm_ = perm; }

 private:
  int perm_of(int i) const { return perm_[static_cast<std::size_t>(i)]; }
  double* row(int i) { return env_.data() + off_[static_cast<std::size_t>(i)] - first_[static_cast<std::size_t>(i)]; }
  const double* row(int i) const {
    return env_.data() + off_[static_cast<std::size_t>(i)] - first_[static_cast<std::size_t>(i)];
  }
  double& at(int i, int j) { return row(i)[j]; }

  int n_;
  std::vector<int> iperm_, perm_, first_;
  std::vector<std::size_t> off_;
  Vec env_;
};

double dot_row(const Row& r, const Vec& x) {
  double s = 0.0;
  for (std::size_t k = 0; k < r.idx.size(); ++k) s += r.val[k] * x[static_cast<std::size_t>(r.idx[k])];
  return s;
}

void axpy_row(const Row& r, double a, Vec& y) {
  for (std::size_t k = 0; k < r.idx.size(); ++k) y[static_cast<std::size_t>(r.idx[k])] += a * r.val[k];
}

// Small dense SPD solve (Cholesky with diagonal safeguard), in place.
void dense_spd_solve(std::vector<double> A, int q, std::vector<double>& b) {
  for (int j = 0; j < q; ++j) {
    double d = A[static_cast<std::size_t>(j * q + j)];
    for (int k = 0; k < j; ++k) d -= A[static_cast<std::size_t>(j * q + k)] * A[static_cast<std::size_t>(j * q + k)];
    d = d > 1e-300 ? std::sqrt(d) : 1e150;
    A[static_cast<std::size_t>(j * q + j)] = d;
    for (int i = j + 1; i < q; ++i) {
      double s = A[static_cast<std::size_t>(i * q + j)];
      for (int k = 0; k < j; ++k) s -= A[static_cast<std::size_t>(i * q + k)] * A[static_cast<std::size_t>(j * q + k)];
      A[static_cast<std::size_t>(i * q + j)] = s / d;
    }
  }
  for (int i = 0; i < q; ++i) {
    double s = b[static_cast<std::size_t>(i)];
    for (int k = 0; k < i; ++k) s -= A[static_cast<std::size_t>(i * q + k)] * b[static_cast<std::size_t>(k)];
    b[static_cast<std::size_t>(i)] = s / A[static_cast<std::size_t>(i * q + i)];
  }
  for (int i = q - 1; i >= 0; --i) {
    double s = b[static_cast<std::size_t>(i)];
    for (int k = i + 1; k < q; ++k) s -= A[static_cast<std::size_t>(k * q + i)] * b[static_cast<std::size_t>(k)];
    b[static_cast<std::size_t>(i)] = s / A[static_cast<std::size_t>(i * q + i)];
  }
}

double max_step(const Vec& v, const Vec& dv) {
  double a = 1.0;
  for (std::size_t i = 0; i < v.size(); ++i)
    if (dv[i] < 0.0) a = std::min(a, -v[i] / dv[i]);
  return a;
}

}  // namespace

Result solve(const Problem& p, const std::vector<double>& x0, double tol, int max_iter) {
  // tol: relative KKT error target (primal residual, dual residual, gap)
  const int n = p.n;
  const int m = static_cast<int>(p.rows.size());
  if (static_cast<int>(p.c.size()) != n || static_cast<int>(x0.size()) != n)
    throw std::invalid_argument("ipm: dimension mismatch");
  std::vector<int> dense_rows;
  for (int r = 0; r < m; ++r)
    if (p.rows[static_cast<std::size_t>(r)].dense) dense_rows.push_back(r);
  const int q = static_cast<int>(dense_rows.size());

  const auto perm = rcm_order(n, p.rows);
  Skyline K(n, p.rows, perm);
  K.set_perm(perm);

  double bnorm = 0.0, cnorm = 0.0;
  for (const auto& r : p.rows) bnorm = std::max(bnorm, std::abs(r.rhs));
  for (double v : p.c) cnorm = std::max(cnorm, std::abs(v));

  Result res;
  Vec x = x0, s(static_cast<std::size_t>(m)), z(static_cast<std::size_t>(m), 1.0);
  for (int r = 0; r < m; ++r) {
    const auto& row = p.rows[static_cast<std::size_t>(r)];
    s[static_cast<std::size_t>(r)] = std::max(dot_row(row, x) - row.rhs, 0.1);
  }
  Vec rp(static_cast<std::size_t>(m)), rd(static_cast<std::size_t>(n)), d(static_cast<std::size_t>(m));
  Vec dx, ds(static_cast<std::size_t>(m)), dz(static_cast<std::size_t>(m));
  Vec dsa(static_cast<std::size_t>(m)), dza(static_cast<std::size_t>(m)), rc(static_cast<std::size_t>(m));
  std::vector<Vec> W(static_cast<std::size_t>(q));
  std::vector<double> C(static_cast<std::size_t>(q * q));
  const double reg = 1e-13;
  double best_err = std::numeric_limits<double>::infinity();
  Vec best_x = x, best_z = z;
  int best_it = 0;

  auto H_apply = [&](const Vec& v, Vec& out) {
    out.assign(static_cast<std::size_t>(n), 0.0);
    for (int r = 0; r < m; ++r) {
      const auto& row = p.rows[static_cast<std::size_t>(r)];
      axpy_row(row, d[static_cast<std::size_t>(r)] * dot_row(row, v), out);
    }
    for (int i = 0; i < n; ++i) out[static_cast<std::size_t>(i)] += reg * v[static_cast<std::size_t>(i)];
  };
  // H^{-1} via K^{-1} and Woodbury over the dense rows
  auto H_solve_once = [&](const Vec& b, Vec& out) {
    K.solve(b, out);
    if (q == 0) return;
    std::vector<double> t(static_cast<std::size_t>(q));
    for (int a = 0; a < q; ++a) t[static_cast<std::size_t>(a)] = dot_row(p.rows[static_cast<std::size_t>(dense_rows[static_cast<std::size_t>(a)])], out);
    dense_spd_solve(C, q, t);
    for (int a = 0; a < q; ++a)
      for (int i = 0; i < n; ++i) out[static_cast<std::size_t>(i)] -= W[static_cast<std::size_t>(a)][static_cast<std::size_t>(i)] * t[static_cast<std::size_t>(a)];
  };
  auto H_solve = [&](const Vec& b, Vec& out) {
    H_solve_once(b, out);
    Vec hx, corr, rr(static_cast<std::size_t>(n));
    for (int ref = 0; ref < 2; ++ref) {  // iterative refinement
      H_apply(out, hx);
      for (int i = 0; i < n; ++i) rr[static_cast<std::size_t>(i)] = b[static_cast<std::size_t>(i)] - hx[static_cast<std::size_t>(i)];
      H_solve_once(rr, corr);
      for (int i = 0; i < n; ++i) out[static_cast<std::size_t>(i)] += corr[static_cast<std::size_t>(i)];
    }
  };
  // direction for a given complementarity target rc
  auto direction = [&](const Vec& rcv, Vec& dxo, Vec& dso, Vec& dzo) {
    Vec rhs(static_cast<std::size_t>(n), 0.0);
    for (int r = 0; r < m; ++r) {
      const double coef = rcv[static_cast<std::size_t>(r)] / s[static_cast<std::size_t>(r)] - d[static_cast<std::size_t>(r)] * rp[static_cast<std::size_t>(r)];
      axpy_row(p.rows[static_cast<std::size_t>(r)], coef, rhs);
    }
    for (int i = 0; i < n; ++i) rhs[static_cast<std::size_t>(i)] -= rd[static_cast<std::size_t>(i)];
    H_solve(rhs, dxo);
    for (int r = 0; r < m; ++r) {
      dso[static_cast<std::size_t>(r)] = dot_row(p.rows[static_cast<std::size_t>(r)], dxo) + rp[static_cast<std::size_t>(r)];
      dzo[static_cast<std::size_t>(r)] = rcv[static_cast<std::size_t>(r)] / s[static_cast<std::size_t>(r)] - d[static_cast<std::size_t>(r)] * dso[static_cast<std::size_t>(r)];
    }
  };

  for (int it = 0; it < max_iter; ++it) {
    double pres = 0.0, dres = 0.0, sz = 0.0;
    for (int r = 0; r < m; ++r) {
      const auto& row = p.rows[static_cast<std::size_t>(r)];
      rp[static_cast<std::size_t>(r)] = dot_row(row, x) - s[static_cast<std::size_t>(r)] - row.rhs;
      pres = std::max(pres, std::abs(rp[static_cast<std::size_t>(r)]));
      sz += s[static_cast<std::size_t>(r)] * z[static_cast<std::size_t>(r)];
    }
    rd = p.c;
    for (int r = 0; r < m; ++r) axpy_row(p.rows[static_cast<std::size_t>(r)], -z[static_cast<std::size_t>(r)], rd);
    for (double v : rd) dres = std::max(dres, std::abs(v));
    const double mu = sz / std::max(1, m);
    double cx = 0.0;
    for (int i = 0; i < n; ++i) cx += p.c[static_cast<std::size_t>(i)] * x[static_cast<std::size_t>(i)];
    res.iterations = it;
    res.primal_residual = pres;
    res.dual_residual = dres;
    res.mu = mu;
    static const bool verbose = std::getenv("PF_IPM_VERBOSE") != nullptr;
    if (verbose) std::fprintf(stderr, "ipm it %d pres %.3e dres %.3e mu %.3e cx %.12g\n", it, pres, dres, mu, cx);
    // relative KKT error; keep the best iterate (late iterations can lose dual
    // accuracy once D = Z/S spans the full double range)
    const double err = std::max({pres / (1.0 + bnorm), dres / (1.0 + cnorm), sz / (1.0 + std::abs(cx))});
    if (err < best_err) {
      best_err = err;
      best_x = x;
      best_z = z;
      best_it = it;
    }
    if (err <= tol) break;
    if (it - best_it > 8 || !std::isfinite(err)) break;
    for (int r = 0; r < m; ++r) d[static_cast<std::size_t>(r)] = z[static_cast<std::size_t>(r)] / s[static_cast<std::size_t>(r)];
    K.clear();
    for (int r = 0; r < m; ++r)
      if (!p.rows[static_cast<std::size_t>(r)].dense) K.add_row(p.rows[static_cast<std::size_t>(r)], d[static_cast<std::size_t>(r)]);
    for (int i = 0; i < n; ++i) K.add_diag(i, reg);
    K.factor();
    if (q > 0) {
      Vec u(static_cast<std::size_t>(n));
      for (int a = 0; a < q; ++a) {
        std::fill(u.begin(), u.end(), 0.0);
        axpy_row(p.rows[static_cast<std::size_t>(dense_rows[static_cast<std::size_t>(a)])], 1.0, u);
        K.solve(u, W[static_cast<std::size_t>(a)]);
      }
      for (int a = 0; a < q; ++a)
        for (int b = 0; b < q; ++b) {
          double v = dot_row(p.rows[static_cast<std::size_t>(dense_rows[static_cast<std::size_t>(a)])], W[static_cast<std::size_t>(b)]);
          if (a == b) v += 1.0 / d[static_cast<std::size_t>(dense_rows[static_cast<std::size_t>(a)])];
          C[static_cast<std::size_t>(a * q + b)] = v;
        }
    }
    // predictor
    for (int r = 0; r < m; ++r) rc[static_cast<std::size_t>(r)] = -s[static_cast<std::size_t>(r)] * z[static_cast<std::size_t>(r)];
    direction(rc, dx, dsa, dza);
    const double ap = max_step(s, dsa), ad = max_step(z, dza);
    double mu_aff = 0.0;
    for (int r = 0; r < m; ++r)
      mu_aff += (s[static_cast<std::size_t>(r)] + ap * dsa[static_cast<std::size_t>(r)]) * (z[static_cast<std::size_t>(r)] + ad * dza[static_cast<std::size_t>(r)]);
    mu_aff /= std::max(1, m);
    const double sigma = std::pow(std::clamp(mu_aff / std::max(mu, 1e-300), 0.0, 1.0), 3.0);
    // corrector
    for (int r = 0; r < m; ++r)
      rc[static_cast<std::size_t>(r)] = -s[static_cast<std::size_t>(r)] * z[static_cast<std::size_t>(r)] + sigma * mu - dsa[static_cast<std::size_t>(r)] * dza[static_cast<std::size_t>(r)];
    direction(rc, dx, ds, dz);
    const double eta = std::max(0.9, 1.0 - 10.0 * mu);
    const double step_p = std::min(1.0, eta * max_step(s, ds));
    const double step_d = std::min(1.0, eta * max_step(z, dz));
    for (int i = 0; i < n; ++i) x[static_cast<std::size_t>(i)] += step_p * dx[static_cast<std::size_t>(i)];
    for (int r = 0; r < m; ++r) {
      s[static_cast<std::size_t>(r)] = std::max(s[static_cast<std::size_t>(r)] + step_p * ds[static_cast<std::size_t>(r)], 1e-300);
      z[static_cast<std::size_t>(r)] = std::max(z[static_cast<std::size_t>(r)] + step_d * dz[static_cast<std::size_t>(r)], 1e-300);
    }
  }
  res.x = best_x;
  res.z = best_z;
  // objective accuracy is far better than the complementarity term once the
  // residuals are tiny; 1e-7 relative KKT error keeps P_d within the parity tolerance
  res.converged = best_err <= std::max(tol, 1e-7);
  res.mu = best_err;
  return res;
}

}  // namespace pipefreeze::ipm
