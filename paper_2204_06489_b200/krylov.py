"""fwi::ConvergenceLog (include/fwi/krylov.hpp:17-33) as Python value types."""
from __future__ import annotations

from dataclasses import dataclass, field


@dataclass
class LogEntryPy:
    iteration: int = 0
    residual_norm: float = 0.0          # true relative residual
    normal_residual: float | None = None
    precond_residual: float | None = None
    wall_time: float = 0.0


@dataclass
class ConvergenceLog:
    entries: list[LogEntryPy] = field(default_factory=list)
    converged: bool = False
    stagnated: bool = False

    def iterations(self) -> int:
        return self.entries[-1].iteration if self.entries else 0

    def final_residual(self) -> float:
        return self.entries[-1].residual_norm if self.entries else 0.0

    def residuals(self):
        return [e.residual_norm for e in self.entries]
