"""Synthetic input series of the benchmark configurations.

Each recipe is deterministic; ``series_sha256`` fingerprints the float64
bytes so the CPU baseline, the golden fixtures and the GPU runs can prove
they saw the same input.
"""

import hashlib
import math
from dataclasses import dataclass

import numpy as np

from .settings import AnalysisSettings

__all__ = ["Workload", "WORKLOADS", "series_sha256", "logistic_series",
           "lorenz_x_series", "sine_noise_series", "uniform_series"]


def series_sha256(values: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(values, np.float64).tobytes()).hexdigest()


def sine_noise_series(length: int = 2000, seed: int = 0) -> np.ndarray:
    """C1: sin over [0, 8 pi] plus 0.25 N(0,1) (tests/helpers.py:13-15 "sine_noise")."""
    rng = np.random.default_rng(seed)
    x = np.linspace(0.0, 8.0 * np.pi, length)
    return np.sin(x) + 0.25 * rng.normal(size=length)


def logistic_series(length: int = 100_000, x0: float = 0.1, burn_in: int = 1000,
                    r: float = 4.0) -> np.ndarray:
    """C2: logistic map x <- r x (1 - x) in Python floats (exact, platform-free)."""
    x = x0
    for _ in range(burn_in):
        x = r * x * (1.0 - x)
    out = np.empty(length)
    for k in range(length):
        x = r * x * (1.0 - x)
        out[k] = x
    return out


def uniform_series(length: int, seed: int) -> np.ndarray:
    """C3/C5: numpy PCG64 uniform [0, 1)."""
    return np.random.default_rng(seed).uniform(0.0, 1.0, length)


def lorenz_x_series(length: int = 500_045, dt: float = 0.01, burn_in: int = 10_000,
                    sigma: float = 10.0, rho: float = 28.0,
                    beta: float = 8.0 / 3.0) -> np.ndarray:
    """C4: x component of the Lorenz system, classical RK4 in Python floats."""
    x, y, z = 1.0, 1.0, 1.0

    def f(x, y, z):
        return sigma * (y - x), x * (rho - z) - y, x * y - beta * z

    out = np.empty(length)
    for k in range(burn_in + length):
        k1 = f(x, y, z)
        k2 = f(x + 0.5 * dt * k1[0], y + 0.5 * dt * k1[1], z + 0.5 * dt * k1[2])
        k3 = f(x + 0.5 * dt * k2[0], y + 0.5 * dt * k2[1], z + 0.5 * dt * k2[2])
        k4 = f(x + dt * k3[0], y + dt * k3[1], z + dt * k3[2])
        x += dt / 6.0 * (k1[0] + 2.0 * k2[0] + 2.0 * k3[0] + k4[0])
        y += dt / 6.0 * (k1[1] + 2.0 * k2[1] + 2.0 * k3[1] + k4[1])
        z += dt / 6.0 * (k1[2] + 2.0 * k2[2] + 2.0 * k3[2] + k4[2])
        if k >= burn_in:
            out[k - burn_in] = x
    return out


def paper_sine_series(length: int = 1_000_001, x_end: float = 1000.0 * math.pi) -> np.ndarray:
    """P: the PyRQA paper's synthetic sine (ingest.py:132-139 generate_sine)."""
    return np.sin(np.linspace(0.0, x_end, length))


@dataclass(frozen=True)
class Workload:
    name: str
    description: str
    make: object           # callable(length) -> np.ndarray
    length: int            # number of samples of the full configuration
    settings: AnalysisSettings

    def series(self, length: int | None = None) -> np.ndarray:
        """The series, or its first ``length`` samples (prefix sample)."""
        full = self.make(self.length)
        return full if length is None else full[:length]

    def n_vectors(self, length: int | None = None) -> int:
        n = self.length if length is None else length
        s = self.settings
        return n - (s.embedding_dimension - 1) * s.time_delay


WORKLOADS = {
    "C1": Workload(
        "C1", "sine+noise N=2,000, m=2, tau=1, L2, r=0.5, Theiler 1",
        lambda n: sine_noise_series(n, 0), 2000,
        AnalysisSettings(2, 1, "euclidean", 0.5, include_main_diagonal=False)),
    "C2": Workload(
        "C2", "logistic map N=100,000, m=3, tau=2, Linf, r=0.05",
        lambda n: logistic_series(n), 100_000,
        AnalysisSettings(3, 2, "maximum", 0.05)),
    "C3": Workload(
        "C3", "uniform random N=1,048,576 vectors, m=3, tau=1, L2, r=0.1",
        lambda n: uniform_series(n, 2024), 2 ** 20 + 2,
        AnalysisSettings(3, 1, "euclidean", 0.1)),
    "C4": Workload(
        "C4", "Lorenz x N=500,000 vectors, m=10, tau=5, L1, r=5.0, Theiler 10",
        lambda n: lorenz_x_series(n), 500_045,
        AnalysisSettings(10, 5, "manhattan", 5.0, include_main_diagonal=False,
                         theiler_corrector=10)),
    "C5": Workload(
        "C5", "uniform random N=4,194,304 vectors, m=3, tau=1, Linf, r=0.1",
        lambda n: uniform_series(n, 2025), 2 ** 22 + 2,
        AnalysisSettings(3, 1, "maximum", 0.1)),
    "P": Workload(
        "P", "paper sine 1,000,001 points over 1000 pi, m=2, tau=2, L2, r=1.0",
        lambda n: paper_sine_series(n), 1_000_001,
        AnalysisSettings(2, 2, "euclidean", 1.0)),
}
