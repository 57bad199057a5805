"""Synthetic scenario configs in the reference's own JSON config schema
(synthgen.cpp:400-489), so the SAME dict drives the reference generator
(workflows::generate_database, used by the oracle) and the device generator
(psg_generate_iterative).

The canonical configs are the ones SURVEY.md §8 defines for BASELINE.json's
configs[0..4]:

* C1  1,000 traces x (64 kernels, 150 iterations, copy)   = 10,050 events/trace
* C2  100,000 traces x (64 kernels, 746 iterations, copy) = 49,982 events/trace
* C3  8,192 ranks x 500 iterations x 64 kernels, GAMESS-like spread
* C4  aurora_like_config with 100 ranks/node (helpers.hpp:117-155)
"""
from __future__ import annotations

import numpy as np

N_KERNELS = 64


def kernel_means(n_kernels: int = N_KERNELS) -> list[float]:
    # mean_time_s = 1e-3 * (1 + k mod 7)
    return [1e-3 * (1 + k % 7) for k in range(n_kernels)]


def ladder_spread(n_ranks: int) -> np.ndarray:
    """Per-rank factors evenly spaced in [0.6, 1.4] (small_iter_config's ladder,
    helpers.hpp:56-57)."""
    r = np.arange(n_ranks, dtype=np.float64)
    return 0.6 + 0.8 * r / max(1, n_ranks - 1)


def gamess_spread(n_ranks: int) -> np.ndarray:
    """One heavy rank at max/mean = 1.5, the rest on an even ladder around a
    mean chosen so the factor mean is exactly 1 (gamess_like_config's shape,
    helpers.hpp:68-112, scaled to n_ranks)."""
    ratio = 1.5
    rest_mean = (n_ranks - ratio) / (n_ranks - 1)
    s = 0.2 * rest_mean
    d = np.linspace(-1.0, 1.0, n_ranks - 1) if n_ranks > 2 else np.zeros(max(0, n_ranks - 1))
    return np.concatenate([[ratio], rest_mean + s * d])


def iterative(n_ranks: int, n_iterations: int, *, n_kernels: int = N_KERNELS,
              spread: str = "ladder", jitter: float = 0.1, copy_segment_s: float = 1e-4,
              seed: int = 1, spread_ranks: int | None = None) -> dict:
    """An iterative scenario.  `spread_ranks` (>= n_ranks) computes the per-rank
    factors for a larger scenario and keeps its first n_ranks, so a prefix of
    ranks is byte-identical to the same ranks of the full scenario (the
    reference draws one stream rank-major)."""
    full = spread_ranks or n_ranks
    f = (ladder_spread if spread == "ladder" else gamess_spread)(full)[:n_ranks]
    means = kernel_means(n_kernels)
    return {
        "type": "iterative",
        "n_ranks": n_ranks,
        "n_iterations": n_iterations,
        "anchor_name": "iter_loop",
        "copy_segment_s": copy_segment_s,
        "hostname": "x1000c0s0b0n0",
        "seed": seed,
        "kernels": [
            {"name": f"gpu_kernel_{k:02d}", "mean_time_s": means[k],
             "across_rank_spread": [float(x) for x in f], "within_rank_jitter_frac": jitter}
            for k in range(n_kernels)
        ],
    }


def c1() -> dict:
    return iterative(1000, 150, seed=1)


def c2(n_ranks: int = 100_000) -> dict:
    return iterative(n_ranks, 746, seed=1, spread_ranks=100_000)


def c3(n_ranks: int = 8192) -> dict:
    return iterative(n_ranks, 500, spread="gamess", seed=3, spread_ranks=8192)


def small(seed: int = 7, n_ranks: int = 4, n_iterations: int = 5, jitter: float = 0.0) -> dict:
    """small_iter_config (helpers.hpp:42-63)."""
    spread = [0.6 + 0.8 * r / max(1, n_ranks - 1) for r in range(n_ranks)]
    return {
        "type": "iterative", "n_ranks": n_ranks, "n_iterations": n_iterations,
        "anchor_name": "solver_loop", "copy_segment_s": 0.004, "seed": seed,
        "kernels": [
            {"name": "kernel_heavy", "mean_time_s": 0.4, "within_rank_jitter_frac": jitter,
             "across_rank_spread": spread},
            {"name": "kernel_light", "mean_time_s": 0.1, "within_rank_jitter_frac": jitter},
        ],
    }


def aurora(ranks_per_node: int = 100, seed: int = 42, jitter: float = 0.02) -> dict:
    """aurora_like_config (helpers.hpp:117-155) with configurable ranks/node;
    C4 uses 100 ranks/node = 100,000 ranks."""
    def site(name, chain, base):
        return {"routine_name": name, "call_chain": chain, "base_time_s": base}
    return {
        "type": "congestion", "n_nodes": 1000, "ranks_per_node": ranks_per_node,
        "rack_id_base": 4000, "chassis_per_rack": 4, "slots_per_chassis": 8,
        "outlier_node_count": 202, "outlier_racks": [4001 + r for r in range(22)],
        "compute_time_s": 2.01, "jitter_frac": jitter, "congestion_multiplier": 4.234375,
        "congested_callsite": 0, "seed": seed,
        "callsites": [
            site("MPI_Allreduce", ["hypre_GMRESSetup", "hypre_BoomerAMGSetup",
                                   "hypre_ParCSRMatrixSetNumNonzeros_core"], 0.64),
            site("MPI_Allreduce", ["hypre_GMRESSolve", "hypre_BoomerAMGSolve"], 0.15),
            site("MPI_Waitall", ["hypre_ParCSRMatrixMatvec"], 0.12),
            site("MPI_Isend", ["hypre_ParCSRCommHandleCreate"], 0.09),
            site("MPI_Irecv", ["hypre_ParCSRCommHandleCreate2"], 0.07),
            site("MPI_Barrier", ["hypre_BoomerAMGCycle"], 0.04),
        ],
    }


def events_per_trace(cfg: dict) -> int:
    return cfg["n_iterations"] * (len(cfg["kernels"]) + 2 + (1 if cfg.get("copy_segment_s", 0) > 0 else 0))


def device_scenario(n_ranks: int, n_iterations: int, *, n_kernels: int = N_KERNELS,
                    spread: str = "ladder", jitter: float = 0.1, copy_segment_s: float = 1e-4,
                    seed: int = 1) -> dict:
    """Compact form of iterative() for the device generator (no per-kernel
    JSON lists; the ladder is shared by every kernel, spread_kernel_stride 0)."""
    f = (ladder_spread if spread == "ladder" else gamess_spread)(n_ranks)
    return {"n_ranks": n_ranks, "n_iterations": n_iterations, "copy_segment_s": copy_segment_s,
            "seed": seed, "device": (np.array(kernel_means(n_kernels), np.float64),
                                     np.full(n_kernels, jitter, np.float64),
                                     np.ascontiguousarray(f, np.float64), 0)}


def c2_device(n_ranks: int = 100_000) -> dict:
    return device_scenario(n_ranks, 746, seed=1)


def device_params(cfg: dict):
    """(mean[k], jitter[k], spread[k][r] or None, stride) for psg_generate_iterative."""
    if "device" in cfg:
        return cfg["device"]
    ks = cfg["kernels"]
    n = cfg["n_ranks"]
    mean = np.array([k["mean_time_s"] for k in ks], dtype=np.float64)
    jit = np.array([k.get("within_rank_jitter_frac", 0.0) for k in ks], dtype=np.float64)
    spreads = [k.get("across_rank_spread", []) for k in ks]
    if all(len(s) == 0 for s in spreads):
        return mean, jit, None, 0
    rows = [np.asarray(s, dtype=np.float64) if len(s) else np.ones(n) for s in spreads]
    if all(np.array_equal(rows[0], r) for r in rows[1:]):
        return mean, jit, np.ascontiguousarray(rows[0]), 0
    return mean, jit, np.ascontiguousarray(np.stack(rows)), n
