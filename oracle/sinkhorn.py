"""Entropic unbalanced OT by Algorithm 1 of the paper — TEST INFRASTRUCTURE ONLY.

Paper notation (Sec. 3.1): discrete measures mu = sum_i mu_i delta_{x_i},
nu = sum_j nu_j delta_{x~_j}; entropy parameter lambda (objective weight 1/lambda,
Def. 2.7, Rem. 2.8 P:223); marginal penalties eta_1, eta_2; cost d^r with r = 2
(the Gaussian Gibbs kernel) or r = 1 (the Laplace Gibbs kernel e^{-lambda ||x - x~||}:
Algorithm 2's input r >= 1, and its r = 1 complexity).

Config notation (BASELINE.json) -> paper (reading R1):
    eps (entropic regularisation)   = 1/lambda
    lam (KL penalty)                = eta_1 = eta_2   (Rem. 3.2)

Algorithm 1, started from gamma^0 = 0 and Delta = 1 (reading R4:
the beta-step comes first).  One "iteration" = one beta-step (3.3) followed by one
gamma-step (3.4), i.e. two kernel sums (reading R2: a fixed iteration count):

    (3.3)  beta_i  <- -eta1/(1+eta1*lambda) * log( sum_j k_ij e^{lambda gamma_j} nu_j )
    (3.4)  gamma_j <- -eta2/(1+eta2*lambda) * log( sum_i k_ij e^{lambda beta_i}  mu_i )

with k_ij = exp(-lambda d_ij^r): exp(-||x_i - x~_j||^2 / eps) for r = 2 and
exp(-||x_i - x~_j|| / eps) for r = 1 (the kernels K^Gauss / K^Lap of (4.2) with l^2 = eps
and l = eps respectively).

The sums are the plain direct kernel sums of ``oracle.direct``.  The plan is
pi_ij = mu_i e^{lambda beta_i} k_ij e^{lambda gamma_j} nu_j.
"""

from dataclasses import dataclass

import numpy as np

from .direct import kernel_sum_direct
from .kernels import GAUSS, LAP, gauss


def gibbs_kind(r):
    """The Gibbs kernel exp(-lambda d^r) as a kernel of (4.2) with parameter eps = 1/lambda:
    K^Gauss (param l^2 = eps) for r = 2, K^Lap (param l = eps) for r = 1."""
    if r == 2:
        return GAUSS
    if r == 1:
        return LAP
    raise ValueError("cost exponent r must be 1 or 2")


def cost_r(d2, r):
    """d^r from the squared distance d^2."""
    return d2 if r == 2 else np.sqrt(d2)


@dataclass
class SinkhornResult:
    beta: np.ndarray
    gamma: np.ndarray
    primal: float
    dual: float
    plan_mass: float
    mass_a: float
    mass_b: float
    max_dbeta: float
    max_dgamma: float
    iters: int


def _xlogy_ratio(p, ref):
    """sum p log(p/ref) with the convention 0 log 0 = 0 (generalised KL)."""
    p = np.asarray(p, dtype=np.float64)
    out = np.zeros_like(p)
    nz = p > 0
    out[nz] = p[nz] * np.log(p[nz] / ref[nz])
    return float(np.sum(out))


def beta_step(x, y, nu, gamma, eps, eta1, r=2):
    """Eq. (3.3): beta_i = -eta1/(1+eta1*lam) log(sum_j k_ij e^{lam gamma_j} nu_j)."""
    lam = 1.0 / eps
    t = kernel_sum_direct(y, np.exp(lam * gamma) * nu, x, gibbs_kind(r), eps)
    return -eta1 / (1.0 + eta1 * lam) * np.log(t)


def gamma_step(x, y, mu, beta, eps, eta2, r=2):
    """Eq. (3.4): gamma_j = -eta2/(1+eta2*lam) log(sum_i k_ij e^{lam beta_i} mu_i)."""
    lam = 1.0 / eps
    tt = kernel_sum_direct(x, np.exp(lam * beta) * mu, y, gibbs_kind(r), eps)
    return -eta2 / (1.0 + eta2 * lam) * np.log(tt)


def plan_marginals(x, mu, y, nu, beta, gamma, eps, r=2):
    """Row/column sums of pi = e^{lam beta} k e^{lam gamma} (.) (mu x nu).

    p_i = sum_j pi_ij,  q_j = sum_i pi_ij, each by one direct kernel sum.
    """
    lam = 1.0 / eps
    t = kernel_sum_direct(y, np.exp(lam * gamma) * nu, x, gibbs_kind(r), eps)
    tt = kernel_sum_direct(x, np.exp(lam * beta) * mu, y, gibbs_kind(r), eps)
    p = mu * np.exp(lam * beta) * t
    q = nu * np.exp(lam * gamma) * tt
    return p, q


def dual_objective(x, mu, y, nu, beta, gamma, eps, eta1, eta2, r=2):
    """The dual function (3.1) of Theorem 3.1, evaluated at (beta, gamma).

    D = -eta1 sum_i e^{-beta_i/eta1} mu_i - eta2 sum_j e^{-gamma_j/eta2} nu_j
        + eta1 sum_i mu_i + eta2 sum_j nu_j
        - (1/lam) sum_ij mu_i (e^{lam beta_i} e^{-lam d_ij^r} e^{lam gamma_j} - 1) nu_j
    The double sum is sum_i mu_i e^{lam beta_i} t_i - mu(X) nu(X), t = K (e^{lam gamma} nu).
    """
    lam = 1.0 / eps
    t = kernel_sum_direct(y, np.exp(lam * gamma) * nu, x, gibbs_kind(r), eps)
    double_sum = float(np.sum(mu * np.exp(lam * beta) * t)) - float(np.sum(mu)) * float(np.sum(nu))
    return (
        -eta1 * float(np.sum(np.exp(-beta / eta1) * mu))
        - eta2 * float(np.sum(np.exp(-gamma / eta2) * nu))
        + eta1 * float(np.sum(mu))
        + eta2 * float(np.sum(nu))
        - double_sum / lam
    )


def primal_objective_dense(x, mu, y, nu, beta, gamma, eps, eta1, eta2, r=2):
    """The discrete primal of (2.9) at the recovered plan, literally as on P:462.

    Builds the n x m plan pi_ij = mu_i e^{lam beta_i} k_ij e^{lam gamma_j} nu_j
    and the cost matrix d_ij^r; small n only.
    """
    lam = 1.0 / eps
    x = np.asarray(x, dtype=np.float64).reshape(len(mu), -1)
    y = np.asarray(y, dtype=np.float64).reshape(len(nu), -1)
    diff = x[:, None, :] - y[None, :, :]
    d2 = np.sum(diff * diff, axis=2)
    dr = cost_r(d2, r)
    k = np.exp(-dr / eps)
    pi = (mu * np.exp(lam * beta))[:, None] * k * (nu * np.exp(lam * gamma))[None, :]
    munu = mu[:, None] * nu[None, :]
    tot = float(np.sum(pi))
    ent = _xlogy_ratio(pi.ravel(), munu.ravel())
    p = np.sum(pi, axis=1)
    q = np.sum(pi, axis=0)
    return (
        float(np.sum(dr * pi))
        + (ent + float(np.sum(munu)) - tot) / lam
        + eta1 * (_xlogy_ratio(p, mu) + float(np.sum(mu)) - tot)
        + eta2 * (_xlogy_ratio(q, nu) + float(np.sum(nu)) - tot)
    )


def primal_objective_marginals(mu, nu, beta, gamma, p, q, eps, eta1, eta2):
    """The same primal rewritten through the plan's marginals only.

    Because log(pi_ij/(mu_i nu_j)) = lam beta_i + lam gamma_j - lam d_ij^2 for the
    plan of P:488, the entropy term (1/lam) sum pi log(pi/(mu nu)) equals
    sum_i beta_i p_i + sum_j gamma_j q_j - <pi, d^r>, so <pi, d^r> cancels (any r):

      P = sum beta p + sum gamma q + (1/lam)(mu(X)nu(X) - pi_tot)
          + eta1 [sum p log(p/mu) + mu(X) - pi_tot] + eta2 [sum q log(q/nu) + nu(X) - pi_tot]

    with pi_tot = sum_i p_i.  ``tests`` pin this against ``primal_objective_dense``.
    """
    lam = 1.0 / eps
    tot = float(np.sum(p))
    ma, mb = float(np.sum(mu)), float(np.sum(nu))
    return (
        float(np.sum(beta * p))
        + float(np.sum(gamma * q))
        + (ma * mb - tot) / lam
        + eta1 * (_xlogy_ratio(p, mu) + ma - tot)
        + eta2 * (_xlogy_ratio(q, nu) + mb - tot)
    )


def uot_sinkhorn_direct(x, mu, y, nu, eps, eta1, eta2=None, iters=100, gamma0=None, stop_tol=0.0,
                        check_every=10, r=2):
    """Algorithm 1 for `iters` iterations from gamma^0 (default 0).

    Returns beta^{2*iters-1}, gamma^{2*iters} and the objective values of the
    recovered plan: primal, dual (3.1), plan mass pi(X x X), and the
    sup-norm changes of the potentials in the last iteration.

    Stopping rule (reading R20 of DESIGN.md; the paper's "while stopping criteria",
    P:502/P:618): with stop_tol > 0, after every `check_every`-th iteration the loop
    ends once max_i |beta_i - beta_i^prev| <= stop_tol and max_j |gamma_j -
    gamma_j^prev| <= stop_tol (changes within that iteration); `iters` is then the cap.

    r: the cost exponent (2: Gaussian Gibbs kernel, 1: Laplace Gibbs kernel).
    """
    if eta2 is None:
        eta2 = eta1
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    mu = np.asarray(mu, dtype=np.float64)
    nu = np.asarray(nu, dtype=np.float64)
    n, m = len(mu), len(nu)
    gamma = np.zeros(m) if gamma0 is None else np.array(gamma0, dtype=np.float64)
    beta = np.zeros(n)
    dbeta = dgamma = 0.0
    done = 0
    for it in range(iters):
        beta_new = beta_step(x, y, nu, gamma, eps, eta1, r)  # Delta odd  (3.3)
        dbeta = float(np.max(np.abs(beta_new - beta))) if n else 0.0
        beta = beta_new
        gamma_new = gamma_step(x, y, mu, beta, eps, eta2, r)  # Delta even (3.4)
        dgamma = float(np.max(np.abs(gamma_new - gamma))) if m else 0.0
        gamma = gamma_new
        done = it + 1
        if stop_tol > 0 and done % check_every == 0 and dbeta <= stop_tol and dgamma <= stop_tol:
            break
    p, q = plan_marginals(x, mu, y, nu, beta, gamma, eps, r)
    primal = primal_objective_marginals(mu, nu, beta, gamma, p, q, eps, eta1, eta2)
    dual = dual_objective(x, mu, y, nu, beta, gamma, eps, eta1, eta2, r)
    return SinkhornResult(
        beta=beta,
        gamma=gamma,
        primal=primal,
        dual=dual,
        plan_mass=float(np.sum(p)),
        mass_a=float(np.sum(mu)),
        mass_b=float(np.sum(nu)),
        max_dbeta=dbeta,
        max_dgamma=dgamma,
        iters=done,
    )


def cstar(x, mu, y, nu, eps, eta1, eta2=None, r=2):
    """Prop. 2.9, Eq. (2.10) with lambda = 1/eps:

        c* = exp(-<mu (x) nu | d^r> / (mu(X) nu(X) (eta1 + eta2 + 1/lambda)))
             * mu(X)^(-eta2 / (eta1 + eta2 + 1/lambda)) * nu(X)^(-eta1 / (...)),

    with <mu (x) nu | d^r> = sum_ij mu_i nu_j ||x_i - x~_j||^r summed by its definition
    (all pairwise differences, numpy pairwise summation)."""
    if eta2 is None:
        eta2 = eta1
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    x = x.reshape(len(mu), -1)
    y = y.reshape(len(nu), -1)
    mu = np.asarray(mu, dtype=np.float64)
    nu = np.asarray(nu, dtype=np.float64)
    total = 0.0
    for i0 in range(0, len(mu), 256):  # blocks of rows only to bound memory
        d2 = np.sum((x[i0:i0 + 256, None, :] - y[None, :, :]) ** 2, axis=2)
        total += float(np.sum(mu[i0:i0 + 256, None] * cost_r(d2, r) * nu[None, :]))
    ma, mb = float(np.sum(mu)), float(np.sum(nu))
    S = eta1 + eta2 + eps
    return float(np.exp(-total / (ma * mb * S)) * ma ** (-eta2 / S) * mb ** (-eta1 / S))


def sinkhorn_divergence_direct(x, mu, y, nu, eps, eta1, eta2=None, iters=100, r=2):
    """The debiased UOT of Eq. (2.12) (Rem. 2.11), lambda = 1/eps:

        sd = UOT(mu, nu) - UOT(mu, mu)/2 - UOT(nu, nu)/2 + (eps/2) (mu(X) - nu(X))^2,

    each UOT the primal value (reading R3) after `iters` iterations of Algorithm 1.
    Returns (sd, (uot_xy, uot_xx, uot_yy))."""
    if eta2 is None:
        eta2 = eta1
    rxy = uot_sinkhorn_direct(x, mu, y, nu, eps, eta1, eta2, iters, r=r)
    rxx = uot_sinkhorn_direct(x, mu, x, mu, eps, eta1, eta2, iters, r=r)
    ryy = uot_sinkhorn_direct(y, nu, y, nu, eps, eta1, eta2, iters, r=r)
    ma, mb = float(np.sum(mu)), float(np.sum(nu))
    sd = rxy.primal - 0.5 * rxx.primal - 0.5 * ryy.primal + 0.5 * eps * (ma - mb) ** 2
    return sd, (rxy.primal, rxx.primal, ryy.primal)


def uot_sinkhorn_scaling_direct(x, mu, y, nu, eps_list, eta1, eta2=None, iters=100, stop_tol=0.0, check_every=10):
    """lambda-scaling (Sec. 5.1.3): Algorithm 1 solved for the entropy
    parameters lambda = 1/eps in the order given (eps decreasing = lambda increasing),
    each stage started from the previous stage's gamma (stage 1 from gamma^0 = 0).
    Returns the last stage's SinkhornResult with `iters` = the total iteration count."""
    gamma0 = None
    total = 0
    r = None
    for eps in eps_list:
        r = uot_sinkhorn_direct(x, mu, y, nu, eps, eta1, eta2, iters, gamma0=gamma0, stop_tol=stop_tol,
                                check_every=check_every)
        total += r.iters
        gamma0 = r.gamma
    r.iters = total
    return r


def transport_cost(x, mu, y, nu, beta, gamma, eps, r=2):
    """<pi, d^r> = sum_ij pi_ij ||x_i - x~_j||^r for the plan of P:488,
    pi_ij = mu_i e^{lam beta_i} k_ij e^{lam gamma_j} nu_j, summed by its definition
    (rows of the dense plan in blocks)."""
    lam = 1.0 / eps
    x = np.asarray(x, dtype=np.float64).reshape(len(mu), -1)
    y = np.asarray(y, dtype=np.float64).reshape(len(nu), -1)
    u = np.asarray(mu) * np.exp(lam * np.asarray(beta))
    v = np.asarray(nu) * np.exp(lam * np.asarray(gamma))
    total = 0.0
    for i0 in range(0, len(mu), 256):
        d2 = np.sum((x[i0:i0 + 256, None, :] - y[None, :, :]) ** 2, axis=2)
        dr = cost_r(d2, r)
        pi = u[i0:i0 + 256, None] * np.exp(-dr / eps) * v[None, :]
        total += float(np.sum(pi * dr))
    return total
