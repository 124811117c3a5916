"""CPU float64 oracle for the FTK hot path (arXiv:1905.12317) -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this package.  The product path (paper_1905_12317_b200) never
imports, links or executes anything here, and this package never imports the
product: the two share no kernels, helpers, tables or constant generators.
The only shared module is synth/ (seeded input generation, no method arithmetic).

Citations: "P:n" = PAPER.md line n (section / equation given beside it).

Modules
  quadrature   radial rule sum_m w_m g(k_m) ~ int_0^K g(k) k dk            (Sec. 3.1)
  fb           Fourier-Bessel coefficients by the periodic trapezoid rule   (Eq. aqkcalc)
  kernel_svd   per-ell operator SVD of J_ell(delta k), two discretizations  (Eq. Jsvd, Remark r:svd P:801-811,
               global relabel + eps truncation                               Eqs. svdtrunc/svdobjective P:822-893)
  ftk          FTK Steps 1-3 literally (Eq. fbk3), cyclic q; log-marginal over the grid
  brute        direct evaluation of the discretized bandlimited inner product (Eq. Xdg P:293-298 with Eq. Fdk)
  closed_form  exact (2 pi)^2 <R_gamma T_delta A, B> for Gaussian-blob images (Eq. planch)
  pixels       pixel images -> polar Fourier samples, the trapezoid sum of Eq. Ahattrap evaluated directly
  bounds       Lemma 2 / Theorem 1 rank bounds, empirical fit, RMS error bound
  ctf          CTF-parameterized kernel (Sec. 6, DESIGN reading R24): the filtered brute force and the
               joint (delta, tau) factorization per ell

Parity status: every function here is pinned by tests in tests/test_oracle_*.py
(see DESIGN.md "Oracle pins"); none is "parity unpinned".
"""
