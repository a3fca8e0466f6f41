// rules.hpp — host scalar rules of the iteration: step-size schedules, adaptive
// step, primal weight and restart decision (stepsize.hpp:31-88,
// solver.hpp:218-235). Pure double arithmetic; the library's host code is
// compiled with -ffp-contract=off, so these are bit-identical to the
// reference's.
#pragma once

#include <cmath>

#include "common.cuh"

namespace rb {

// stepsize.hpp:31-42
inline rapdhg_step_params step_schedule_theoretical(int k, int horizon, double norm_q,
                                                    double norm_a) {
  if (horizon < 1) invalid("step schedule: horizon must be >= 1");
  if (k < 0 || k >= horizon) invalid("step schedule: k out of range");
  if (norm_a <= 0.0) norm_a = norm_q / horizon;
  if (norm_a <= 0.0) invalid("step schedule: both norms are zero");
  rapdhg_step_params sp;
  sp.beta = 0.5 * (k + 2);
  sp.theta = static_cast<double>(k) / (k + 1);
  sp.eta = (k + 1) / (2.0 * (norm_q + horizon * norm_a));
  sp.tau = (k + 1) / (2.0 * horizon * norm_a);
  return sp;
}

// stepsize.hpp:47-54
inline rapdhg_step_params pdhg_constant_steps(double norm_q, double norm_a) {
  if (norm_a <= 0.0) {
    if (norm_q <= 0.0) invalid("pdhg steps: both norms are zero");
    return rapdhg_step_params{1.0, 1.0, 1.0 / norm_q, 0.0};
  }
  return rapdhg_step_params{1.0, 1.0, 1.0 / (norm_q + 2.0 * norm_a), 1.0 / (2.0 * norm_a)};
}

// stepsize.hpp:59-68
inline double adaptive_eta(int k, double prev_eta, double norm_q, double norm_a, double omega) {
  if (omega <= 0.0) invalid("adaptive_eta: omega must be positive");
  if (norm_q <= 0.0 && norm_a <= 0.0) invalid("adaptive_eta: both norms are zero");
  const double qw = norm_q / omega;
  if (k == 0) return 1.98 / (qw + std::sqrt(4.0 * norm_a * norm_a + qw * qw));
  const double fresh =
      0.99 * (k + 2) / (qw + std::sqrt(norm_a * norm_a * (k + 2.0) * (k + 2.0) + qw * qw));
  const double grow = (1.0 + 1.0 / k) * prev_eta;
  return (fresh < grow) ? fresh : grow;  // std::min(grow, fresh)
}

constexpr double kZeroNormTol = 1e-10;

// stepsize.hpp:73-78 (norms computed on the device)
inline double primal_weight_init(double norm_c, double norm_b) {
  if (norm_c > kZeroNormTol && norm_b > kZeroNormTol) return norm_c / norm_b;
  return 1.0;
}

// stepsize.hpp:83-88
inline double primal_weight_update(double delta_x, double delta_y, double omega_prev) {
  if (omega_prev <= 0.0) invalid("primal weight must be positive");
  if (delta_x <= kZeroNormTol || delta_y <= kZeroNormTol) return omega_prev;
  constexpr double kTheta = 0.2;
  return std::exp(kTheta * std::log(delta_y / delta_x) + (1.0 - kTheta) * std::log(omega_prev));
}

// solver.hpp:214-235
inline bool restart_decision(int policy, double cand, double cand_prev, double start, long k,
                             long total_iters, long fixed_length) {
  switch (policy) {
    case RAPDHG_RESTART_NONE: return false;
    case RAPDHG_RESTART_FIXED: return k >= fixed_length;
    case RAPDHG_RESTART_HALVING: return cand <= 0.5 * start;
    case RAPDHG_RESTART_PDQP:
      if (cand <= 0.2 * start) return true;
      if (cand <= 0.8 * start && cand > cand_prev) return true;
      return k >= 0.36 * static_cast<double>(total_iters);
  }
  return false;
}

// SolverConfig::validate (solver.hpp:57-63)
inline void validate_config(const rapdhg_config& c) {
  if (c.tol <= 0.0) invalid("tol must be positive");
  if (c.restart == RAPDHG_RESTART_FIXED && c.restart_length < 1)
    invalid("fixed restart requires restart_length >= 1");
  if (c.check_interval < 1) invalid("check_interval must be >= 1");
  if (c.max_iters < 0) invalid("max_iters must be >= 0");
}

}  // namespace rb
