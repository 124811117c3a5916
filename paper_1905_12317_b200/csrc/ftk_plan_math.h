// Host-side plan mathematics (double precision, untimed; "planning stage").
#pragma once
#include <complex>
#include <string>
#include <vector>

namespace ftk {

// Gauss-Legendre on [-1,1] by Newton on P_n (nodes ascending).
void gauss_legendre(int n, std::vector<double>& t, std::vector<double>& w);
// Gauss-Jacobi(alpha, beta) on [-1,1], weight (1-t)^alpha (1+t)^beta, by Golub-Welsch (nodes ascending).
bool gauss_jacobi(int n, double alpha, double beta, std::vector<double>& t, std::vector<double>& w);
// J_0..J_nmax at x >= 0 by Miller's backward recurrence normalized with J_0 + 2 sum J_2k = 1.
void bessel_j_all(double x, int nmax, double* out);
// Radial rule of the plan (reading R2): 0 = Gauss-Legendre x k dk, 1 = Gauss-Jacobi(0,1) on
// [0, k_max]; sum w = k_max^2 / 2.  false if the Golub-Welsch iteration fails.
bool radial_rule_nodes(int n_k, double k_max, int rule, std::vector<double>& k, std::vector<double>& w);
// One-sided (Hestenes) Jacobi SVD of a column-major m x n matrix A (m >= n): A = U diag(S) V^T,
// singular values descending.  A is overwritten by U (columns); V is n x n column-major.
bool svd_jacobi(int m, int n, std::vector<double>& A, std::vector<double>& S, std::vector<double>& V);

struct Term {
  int ell;      // signed Bessel order
  int eta;      // 0-based index in the ell block
  double sigma;
};

struct PlanMath {
  // inputs
  int n = 0, n_k = 0, n_psi = 0, N_t = 0, rule = 0, svd_nodes = 96;
  double K_cycles = 0, k_max = 0, delta_max = 0, W = 0, eps = 0;
  std::vector<double> shifts;           // [N_t][2]
  // CTF-parameterized kernel (Sec. 6 "Other 2D kernels"; reading R24): n_tau > 0
  // radial filters c_tau(k_m) ([n_tau][n_k], on this plan's radial nodes); the shift list then holds
  // n_tau copies of the N_base user shifts (virtual shift v = tau * N_base + t) and the factorization is
  // F(delta, k) c_tau(|k|) = sum_zeta Y_zeta(delta, tau) G_zeta(k).
  int n_tau = 0, N_base = 0;
  std::vector<double> filt;
  // outputs
  std::vector<double> k, w;             // radial rule
  std::vector<Term> terms;              // zeta order, both signs
  std::vector<double> G;                // [H][n_k]  Sigma V(k_m)
  std::vector<std::complex<double>> Y;  // [N_t][H]  U(|delta|) e^{-i ell (omega + pi/2)}
  std::vector<std::vector<double>> sigma_all;  // per ell >= 0, all computed singular values
  int H = 0, H_plus = 0, H0 = 0, K3 = 0, ell_max = 0;
  double certificate = 0;
  std::string error;
  // returns 0 on success, FTK status otherwise (error filled)
  int build();
};

}  // namespace ftk
