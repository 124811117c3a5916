// Host plan mathematics for the FTK hot path (double precision, untimed).
//
// PAPER.md Sec. 4.5 (Eq. Jsvd, Remark r:svd P:801-811, Eq. svdtrunc P:822-831,
// relabel + eps truncation P:858-873).  The operator SVD of J_ell(delta k) on [0,D] x [0,K] with
// weights delta d delta, k dk is computed in the rescaled variables of the Lemma 2 proof
// (P:1029-1032): x = K delta in [0, 2 pi W], y = k / K in [0, 1].  Discretization: symmetric
// Nystrom on Gauss-Jacobi(0,1) nodes (weight x dx resp. y dy), dense one-sided Jacobi SVD, Nystrom
// extension off the nodes.  (The CPU oracle uses its own scipy/numpy code; nothing is shared.)
#include "ftk_plan_math.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <numeric>

#include "../../include/ftk.h"

namespace ftk {

static const double kPi = 3.14159265358979323846;

void gauss_legendre(int n, std::vector<double>& t, std::vector<double>& w) {
  t.assign(n, 0.0);
  w.assign(n, 0.0);
  for (int i = 0; i < n; ++i) {
    double x = std::cos(kPi * (i + 0.75) / (n + 0.5));
    double dp = 1.0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = x;
      for (int k = 2; k <= n; ++k) {
        double p2 = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      if (n == 1) { p1 = x; p0 = 1.0; }
      dp = n * (x * p1 - p0) / (x * x - 1.0);
      double dx = p1 / dp;
      x -= dx;
      if (std::fabs(dx) < 1e-16) {
        // one more evaluation of dp at the converged node
        double q0 = 1.0, q1 = x;
        for (int k = 2; k <= n; ++k) {
          double q2 = ((2.0 * k - 1.0) * x * q1 - (k - 1.0) * q0) / k;
          q0 = q1;
          q1 = q2;
        }
        if (n == 1) { q1 = x; q0 = 1.0; }
        dp = n * (x * q1 - q0) / (x * x - 1.0);
        break;
      }
    }
    t[n - 1 - i] = x;
    w[n - 1 - i] = 2.0 / ((1.0 - x * x) * dp * dp);
  }
}

// Symmetric tridiagonal implicit QL with eigenvectors (z: n x n row-major, z[r*n+c]).  Source: the textbook
// implicit-shift QL iteration of the EISPACK tql2 lineage as given in Press et al., Numerical Recipes, 2nd ed.,
// Sec. 11.3 ("tqli"), with its temporaries (f, g, r, s, c, p, b); host-side plan setup only (untimed).
static bool tridiag_ql(int n, std::vector<double>& d, std::vector<double>& e, std::vector<double>& z) {
  for (int i = 1; i < n; ++i) e[i - 1] = e[i];
  e[n - 1] = 0.0;
  for (int l = 0; l < n; ++l) {
    int iter = 0, m;
    do {
      for (m = l; m < n - 1; ++m) {
        double dd = std::fabs(d[m]) + std::fabs(d[m + 1]);
        if (std::fabs(e[m]) <= 1e-17 * dd) break;
      }
      if (m != l) {
        if (iter++ == 100) return false;
        double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
        double r = std::hypot(g, 1.0);
        g = d[m] - d[l] + e[l] / (g + std::copysign(r, g));
        double s = 1.0, c = 1.0, p = 0.0;
        int i;
        for (i = m - 1; i >= l; --i) {
          double f = s * e[i], b = c * e[i];
          e[i + 1] = (r = std::hypot(f, g));
          if (r == 0.0) {
            d[i + 1] -= p;
            e[m] = 0.0;
            break;
          }
          s = f / r;
          c = g / r;
          g = d[i + 1] - p;
          r = (d[i] - g) * s + 2.0 * c * b;
          d[i + 1] = g + (p = s * r);
          g = c * r - b;
          for (int k = 0; k < n; ++k) {
            f = z[k * n + i + 1];
            z[k * n + i + 1] = s * z[k * n + i] + c * f;
            z[k * n + i] = c * z[k * n + i] - s * f;
          }
        }
        if (r == 0.0 && i >= l) continue;
        d[l] -= p;
        e[l] = g;
        e[m] = 0.0;
      }
    } while (m != l);
  }
  return true;
}

bool gauss_jacobi(int n, double alpha, double beta, std::vector<double>& t, std::vector<double>& w) {
  std::vector<double> d(n), e(n, 0.0), z((size_t)n * n, 0.0);
  const double ab = alpha + beta;
  for (int k = 0; k < n; ++k) {
    d[k] = (k == 0) ? (beta - alpha) / (ab + 2.0)
                    : (beta * beta - alpha * alpha) / ((2.0 * k + ab) * (2.0 * k + ab + 2.0));
    if (k >= 1) {
      double num = 4.0 * k * (k + alpha) * (k + beta) * (k + ab);
      double den = (2.0 * k + ab) * (2.0 * k + ab) * (2.0 * k + ab + 1.0) * (2.0 * k + ab - 1.0);
      e[k] = std::sqrt(num / den);
    }
    z[(size_t)k * n + k] = 1.0;
  }
  if (!tridiag_ql(n, d, e, z)) return false;
  const double mu0 = std::pow(2.0, ab + 1.0) * std::tgamma(alpha + 1.0) * std::tgamma(beta + 1.0) / std::tgamma(ab + 2.0);
  std::vector<int> idx(n);
  std::iota(idx.begin(), idx.end(), 0);
  std::sort(idx.begin(), idx.end(), [&](int a, int b) { return d[a] < d[b]; });
  t.resize(n);
  w.resize(n);
  for (int i = 0; i < n; ++i) {
    t[i] = d[idx[i]];
    double z0 = z[idx[i]];  // first component of eigenvector idx[i] (row 0)
    w[i] = mu0 * z0 * z0;
  }
  return true;
}

void bessel_j_all(double x, int nmax, double* J) {
  for (int i = 0; i <= nmax; ++i) J[i] = 0.0;
  if (x == 0.0) {
    J[0] = 1.0;
    return;
  }
  const int big = std::max(nmax, (int)x);
  // Miller start index: the even N above max(nmax, x) + sqrt(ACC (big + 1)) with ACC = 40, the heuristic of
  // Numerical Recipes' bessj (2nd ed., Sec. 6.5)
  int N = 2 * ((big + 40 + (int)std::sqrt(40.0 * (big + 1))) / 2);
  double bjp = 0.0, bj = 1.0, sum = 0.0;
  for (int kk = N; kk > 0; --kk) {
    double bjm = (2.0 * kk / x) * bj - bjp;
    bjp = bj;
    bj = bjm;
    const int m = kk - 1;
    if (std::fabs(bj) > 1e200) {
      bj *= 1e-200;
      bjp *= 1e-200;
      sum *= 1e-200;
      for (int i = m + 1; i <= nmax; ++i) J[i] *= 1e-200;
    }
    if (m <= nmax) J[m] = bj;
    if (m > 0 && (m % 2) == 0) sum += 2.0 * bj;
  }
  sum += bj;  // J_0
  const double inv = 1.0 / sum;
  for (int i = 0; i <= nmax; ++i) J[i] *= inv;
}

bool svd_jacobi(int m, int n, std::vector<double>& A, std::vector<double>& S, std::vector<double>& V) {
  V.assign((size_t)n * n, 0.0);
  for (int i = 0; i < n; ++i) V[(size_t)i * n + i] = 1.0;
  double fro2 = 0;
  for (double x : A) fro2 += x * x;
  // pairs whose coupling is below this absolute level only affect singular values < ~1e-16 ||A||_F
  const double tiny = 1e-32 * fro2;
  bool conv = false;
  for (int sweep = 0; sweep < 80 && !conv; ++sweep) {
    int rot = 0;
    for (int p = 0; p < n - 1; ++p) {
      double* ap = &A[(size_t)p * m];
      for (int q = p + 1; q < n; ++q) {
        double* aq = &A[(size_t)q * m];
        double al = 0, be = 0, ga = 0;
        for (int i = 0; i < m; ++i) {
          al += ap[i] * ap[i];
          be += aq[i] * aq[i];
          ga += ap[i] * aq[i];
        }
        if (al == 0.0 || be == 0.0 || std::fabs(ga) <= 1e-15 * std::sqrt(al * be) || std::fabs(ga) <= tiny) continue;
        ++rot;
        double zeta = (be - al) / (2.0 * ga);
        double t = (zeta >= 0 ? 1.0 : -1.0) / (std::fabs(zeta) + std::sqrt(1.0 + zeta * zeta));
        double c = 1.0 / std::sqrt(1.0 + t * t), s = c * t;
        for (int i = 0; i < m; ++i) {
          double x = ap[i], y = aq[i];
          ap[i] = c * x - s * y;
          aq[i] = s * x + c * y;
        }
        double* vp = &V[(size_t)p * n];
        double* vq = &V[(size_t)q * n];
        for (int i = 0; i < n; ++i) {
          double x = vp[i], y = vq[i];
          vp[i] = c * x - s * y;
          vq[i] = s * x + c * y;
        }
      }
    }
    conv = (rot == 0);
  }
  std::vector<double> s(n);
  for (int j = 0; j < n; ++j) {
    double acc = 0;
    for (int i = 0; i < m; ++i) acc += A[(size_t)j * m + i] * A[(size_t)j * m + i];
    s[j] = std::sqrt(acc);
  }
  std::vector<int> idx(n);
  std::iota(idx.begin(), idx.end(), 0);
  std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return s[a] > s[b]; });
  std::vector<double> U2((size_t)m * n), V2((size_t)n * n);
  S.resize(n);
  for (int j = 0; j < n; ++j) {
    const int o = idx[j];
    S[j] = s[o];
    const double inv = s[o] > 0 ? 1.0 / s[o] : 0.0;
    for (int i = 0; i < m; ++i) U2[(size_t)j * m + i] = A[(size_t)o * m + i] * inv;
    for (int i = 0; i < n; ++i) V2[(size_t)j * n + i] = V[(size_t)o * n + i];
  }
  A.swap(U2);
  V.swap(V2);
  return conv;
}

bool radial_rule_nodes(int n_k, double k_max, int rule, std::vector<double>& k, std::vector<double>& w) {
  std::vector<double> t, om;
  if (rule == 0) {
    gauss_legendre(n_k, t, om);
  } else if (!gauss_jacobi(n_k, 0.0, 1.0, t, om)) {
    return false;
  }
  k.resize(n_k);
  w.resize(n_k);
  for (int m = 0; m < n_k; ++m) {
    k[m] = 0.5 * k_max * (1.0 + t[m]);
    w[m] = rule == 0 ? om[m] * 0.5 * k_max * k[m] : om[m] * 0.25 * k_max * k_max;
  }
  return true;
}

namespace {
struct Kept {
  int ell, eta;
  double sigma;
  std::vector<double> Ux;  // U column on x nodes (orthonormal vector entries)
  std::vector<double> Vy;  // V column on y nodes
};
}  // namespace

int PlanMath::build() {
  if (n <= 0 || K_cycles <= 0 || n_k <= 0 || n_psi <= 0 || N_t <= 0 || !(eps > 0 && eps < 1) || !(delta_max > 0)) {
    error = "ftk_plan_create: need n > 0, K > 0, n_k > 0, n_psi > 0, N_t > 0, 0 < eps < 1, delta_max > 0";
    return FTK_EINVAL;
  }
  if ((int)shifts.size() != 2 * N_t) {
    error = "ftk_plan_create: shift list size mismatch";
    return FTK_EINVAL;
  }
  for (int t = 0; t < N_t; ++t) {
    double d = std::hypot(shifts[2 * t], shifts[2 * t + 1]);
    if (!(d <= delta_max * (1.0 + 1e-12))) {
      char buf[160];
      std::snprintf(buf, sizeof buf, "shift %d (%.6g, %.6g) has |delta| = %.9g > delta_max = %.9g", t,
                    shifts[2 * t], shifts[2 * t + 1], d, delta_max);
      error = buf;
      return FTK_ERANGE;
    }
  }
  k_max = 2.0 * kPi * K_cycles / n;  // reading R1: K in cycles per image width
  W = delta_max * k_max / (2.0 * kPi);
  const double a = 2.0 * kPi * W;

  // ---- radial rule
  if (!radial_rule_nodes(n_k, k_max, rule, k, w)) {
    error = "Gauss-Jacobi radial rule: QL iteration failed";
    return FTK_ENUMERIC;
  }
  {
    double sw = 0;
    for (double x : w) sw += x;
    if (std::fabs(sw - 0.5 * k_max * k_max) > 1e-11 * k_max * k_max) {
      error = "radial rule self-check failed: sum w != K^2/2";
      return FTK_ENUMERIC;
    }
  }

  const bool ctf = n_tau > 0;
  if (ctf && ((int)filt.size() != n_tau * n_k || N_base <= 0 || N_base * n_tau != N_t)) {
    error = "ftk_plan_create_ctf: filter table / shift list size mismatch";
    return FTK_EINVAL;
  }
  for (double x : filt)
    if (!std::isfinite(x)) {
      error = "ftk_plan_create_ctf: non-finite filter value";
      return FTK_EINVAL;
    }

  // ---- Nystrom nodes (Gauss-Jacobi(0,1) on [0,a] and [0,1]).  CTF mode: the k side is the radial
  // rule itself (the filters are known only on k_m), so the x side needs N n_tau >= n_k rows.
  const int N = ctf ? std::max(svd_nodes, (n_k + n_tau - 1) / n_tau) : svd_nodes;
  std::vector<double> tj, oj;
  if (!gauss_jacobi(N, 0.0, 1.0, tj, oj)) {
    error = "Gauss-Jacobi Nystrom nodes: QL iteration failed";
    return FTK_ENUMERIC;
  }
  std::vector<double> xs(N), wx(N), ys(N), wy(N), swx(N), swy(N);
  for (int i = 0; i < N; ++i) {
    xs[i] = 0.5 * a * (1.0 + tj[i]);
    wx[i] = oj[i] * 0.25 * a * a;
    ys[i] = 0.5 * (1.0 + tj[i]);
    wy[i] = oj[i] * 0.25;
    swx[i] = std::sqrt(wx[i]);
    swy[i] = std::sqrt(wy[i]);
  }
  const double calH = std::max(kPi * std::exp(2.0) * W, std::log(2.0 * kPi * W / eps)) + 1.5;  // Theorem 1
  const int Lc = std::min(400, (int)std::ceil(2.0 * calH));
  // CTF mode: y_m = k_m / K with weights w_m / K^2 (the same y dy measure, sum 1/2); rows (x_i, tau)
  // with weight 1 per tau, so the discarded tail bounds every filter's error (reading R24).
  const int NY = ctf ? n_k : N;
  const int NR = ctf ? N * n_tau : N;
  std::vector<double> ymv(NY), symv(NY);
  for (int j = 0; j < NY; ++j) {
    ymv[j] = ctf ? k[j] / k_max : ys[j];
    symv[j] = ctf ? std::sqrt(w[j]) / k_max : swy[j];
  }
  std::vector<double> Jtab((size_t)N * NY * (Lc + 1));
  for (int i = 0; i < N; ++i)
    for (int j = 0; j < NY; ++j) bessel_j_all(xs[i] * ymv[j], Lc, &Jtab[((size_t)i * NY + j) * (Lc + 1)]);

  std::vector<Kept> kept;
  sigma_all.clear();
  for (int ell = 0; ell <= Lc; ++ell) {
    std::vector<double> M((size_t)NR * NY), S, Vm;
    for (int j = 0; j < NY; ++j)
      for (int r = 0; r < NR; ++r) {
        const int i = r % N, ta = r / N;
        const double cf = ctf ? filt[(size_t)ta * n_k + j] : 1.0;
        M[(size_t)j * NR + r] = swx[i] * Jtab[((size_t)i * NY + j) * (Lc + 1) + ell] * cf * symv[j];
      }
    if (!svd_jacobi(NR, NY, M, S, Vm)) {
      error = "one-sided Jacobi SVD did not converge";
      return FTK_ENUMERIC;
    }
    for (double s : S)
      if (!std::isfinite(s)) {
        error = "non-finite singular value";
        return FTK_ENUMERIC;
      }
    sigma_all.push_back(S);
    int nk = 0;
    for (int e = 0; e < NY; ++e) {
      if (!(S[e] > eps)) break;
      ++nk;
      Kept kp;
      kp.ell = ell;
      kp.eta = e;
      kp.sigma = S[e];
      kp.Ux.assign(&M[(size_t)e * NR], &M[(size_t)e * NR] + NR);
      kp.Vy.assign(&Vm[(size_t)e * NY], &Vm[(size_t)e * NY] + NY);
      // sign convention: largest-|v| node value positive (products U Sigma V are sign-free)
      int jm = 0;
      double best = -1;
      for (int j = 0; j < NY; ++j) {
        double v = std::fabs(kp.Vy[j] / symv[j]);
        if (v > best) { best = v; jm = j; }
      }
      if (kp.Vy[jm] < 0) {
        for (double& x : kp.Ux) x = -x;
        for (double& x : kp.Vy) x = -x;
      }
      kept.push_back(std::move(kp));
    }
    if (ell >= 1 && nk == 0 && ell > a) break;  // H_ell non-increasing beyond the turning region
  }
  if (kept.empty()) {
    error = "no singular value exceeds eps";
    return FTK_ENUMERIC;
  }

  // ---- terms, both signs, zeta order (reading R8)
  terms.clear();
  for (const auto& kp : kept) {
    terms.push_back({kp.ell, kp.eta, kp.sigma});
    if (kp.ell > 0) terms.push_back({-kp.ell, kp.eta, kp.sigma});
  }
  std::stable_sort(terms.begin(), terms.end(), [](const Term& p, const Term& q) {
    if (p.sigma != q.sigma) return p.sigma > q.sigma;
    if (std::abs(p.ell) != std::abs(q.ell)) return std::abs(p.ell) < std::abs(q.ell);
    if ((p.ell > 0) != (q.ell > 0)) return p.ell > 0;
    return p.eta < q.eta;
  });
  H = (int)terms.size();
  H_plus = H0 = ell_max = 0;
  for (const auto& tm : terms) {
    if (tm.ell >= 0) ++H_plus;
    if (tm.ell == 0) ++H0;
    ell_max = std::max(ell_max, std::abs(tm.ell));
  }
  K3 = 2 * H_plus - H0;

  // ---- Nystrom extension: u(x) = (1/s) sum_j sqrt(wy_j) J(x y_j) V_j ; v(y) = (1/s) sum_i sqrt(wx_i) J(x_i y) U_i
  auto find_kept = [&](int ell, int eta) -> const Kept& {
    for (const auto& kp : kept)
      if (kp.ell == ell && kp.eta == eta) return kp;
    return kept[0];
  };
  // v at y_m = k_m / k_max
  std::vector<double> Jb(ell_max + 1);
  const int NJ = ctf ? 0 : N;  // plain-mode Nystrom tables only
  std::vector<double> Jym((size_t)n_k * NJ * (ell_max + 1));
  for (int m = 0; m < n_k; ++m)
    for (int i = 0; i < NJ; ++i) bessel_j_all(xs[i] * (k[m] / k_max), ell_max, &Jym[((size_t)m * N + i) * (ell_max + 1)]);
  std::vector<double> Jxt((size_t)N_t * NJ * (ell_max + 1));
  std::vector<double> dd(N_t), ww(N_t);
  for (int tt = 0; tt < N_t; ++tt) {
    dd[tt] = std::hypot(shifts[2 * tt], shifts[2 * tt + 1]);
    ww[tt] = std::atan2(shifts[2 * tt + 1], shifts[2 * tt]);
    for (int j = 0; j < NJ; ++j) bessel_j_all(k_max * dd[tt] * ys[j], ell_max, &Jxt[((size_t)tt * N + j) * (ell_max + 1)]);
  }
  G.assign((size_t)H * n_k, 0.0);
  Y.assign((size_t)N_t * H, 0.0);
  if (ctf) {
    // k side: v(y_m) = V_m / sqrt(wy_m) directly on the radial nodes; (delta, tau) side by the Nystrom
    // extension u(x, tau) = (1/s) sum_m J_ell(x y_m) c_tau(k_m) sqrt(wy_m) V_m at x = K |delta_t|.
    std::vector<double> Jt((size_t)N_base * n_k * (ell_max + 1));
    for (int tt = 0; tt < N_base; ++tt)
      for (int m = 0; m < n_k; ++m) bessel_j_all(k_max * dd[tt] * ymv[m], ell_max, &Jt[((size_t)tt * n_k + m) * (ell_max + 1)]);
    for (int z = 0; z < H; ++z) {
      const Term& tm = terms[z];
      const int L = std::abs(tm.ell);
      const Kept& kp = find_kept(L, tm.eta);
      const double par = (tm.ell < 0 && (L & 1)) ? -1.0 : 1.0;
      for (int m = 0; m < n_k; ++m) G[(size_t)z * n_k + m] = tm.sigma * par * (kp.Vy[m] / symv[m]) / k_max;
      for (int tt = 0; tt < N_t; ++tt) {
        const int tb = tt % N_base, ta = tt / N_base;
        double acc = 0;
        for (int m = 0; m < n_k; ++m)
          acc += Jt[((size_t)tb * n_k + m) * (ell_max + 1) + L] * filt[(size_t)ta * n_k + m] * symv[m] * kp.Vy[m];
        const double U = k_max * acc / kp.sigma;
        const double ph = -tm.ell * (ww[tt] + 0.5 * kPi);
        Y[(size_t)tt * H + z] = std::complex<double>(U * std::cos(ph), U * std::sin(ph));
      }
    }
  }
  for (int z = 0; z < (ctf ? 0 : H); ++z) {
    const Term& tm = terms[z];
    const int L = std::abs(tm.ell);
    const Kept& kp = find_kept(L, tm.eta);
    const double par = (tm.ell < 0 && (L & 1)) ? -1.0 : 1.0;  // J_{-l} = (-1)^l J_l
    for (int m = 0; m < n_k; ++m) {
      double acc = 0;
      for (int i = 0; i < N; ++i) acc += swx[i] * Jym[((size_t)m * N + i) * (ell_max + 1) + L] * kp.Ux[i];
      const double v = acc / kp.sigma;
      G[(size_t)z * n_k + m] = tm.sigma * par * v / k_max;  // G = Sigma V(k), V(k) = v(k/K)/K
    }
    for (int tt = 0; tt < N_t; ++tt) {
      double acc = 0;
      for (int j = 0; j < N; ++j) acc += swy[j] * Jxt[((size_t)tt * N + j) * (ell_max + 1) + L] * kp.Vy[j];
      const double U = k_max * acc / kp.sigma;  // U(delta) = K u(K delta)
      const double ph = -tm.ell * (ww[tt] + 0.5 * kPi);
      Y[(size_t)tt * H + z] = std::complex<double>(U * std::cos(ph), U * std::sin(ph));
    }
  }

  // ---- certificate: max |F - F^SVD| over the 64 largest shifts x all k_m x all psi_p
  {
    std::vector<int> order(N_t);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int p, int q) { return dd[p] > dd[q]; });
    const int ns = std::min(N_t, 64);
    std::vector<std::complex<double>> eil((size_t)(2 * ell_max + 1) * n_psi);
    for (int l = -ell_max; l <= ell_max; ++l)
      for (int p = 0; p < n_psi; ++p) {
        double ph = l * 2.0 * kPi * p / n_psi;
        eil[(size_t)(l + ell_max) * n_psi + p] = std::complex<double>(std::cos(ph), std::sin(ph));
      }
    double worst = 0;
    std::vector<std::complex<double>> c(2 * ell_max + 1);
    for (int s = 0; s < ns; ++s) {
      const int tt = order[s];
      for (int m = 0; m < n_k; ++m) {
        std::fill(c.begin(), c.end(), std::complex<double>(0, 0));
        for (int z = 0; z < H; ++z) c[terms[z].ell + ell_max] += Y[(size_t)tt * H + z] * G[(size_t)z * n_k + m];
        for (int p = 0; p < n_psi; ++p) {
          std::complex<double> fs(0, 0);
          for (int l = 0; l <= 2 * ell_max; ++l) fs += c[l] * eil[(size_t)l * n_psi + p];
          const double psi = 2.0 * kPi * p / n_psi;
          const double ph = -k[m] * (shifts[2 * tt] * std::cos(psi) + shifts[2 * tt + 1] * std::sin(psi));
          const double cf = ctf ? filt[(size_t)(tt / N_base) * n_k + m] : 1.0;
          worst = std::max(worst, std::abs(cf * std::complex<double>(std::cos(ph), std::sin(ph)) - fs));
        }
      }
    }
    certificate = worst;
  }
  return FTK_OK;
}

}  // namespace ftk
