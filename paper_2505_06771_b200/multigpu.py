"""Multi-GPU plumbing: one process per GPU, independent contiguous env slices.

There is no exchange in the step (envs are independent); the only
collective is the final reduction of the per-device episode statistics
(mrsim_get_stats partials; EpisodeStats / RunSummary, harness.hpp:157-194).
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    envs_per_rank: int

    @property
    def first_episode(self) -> int:
        """Episode index of this rank's env 0 (harness wave seeding, harness.hpp:227-232)."""
        return self.rank * self.envs_per_rank

    @property
    def episode_stride(self) -> int:
        """Auto-reset advances every env slot by the global batch size."""
        return self.world * self.envs_per_rank

    def global_env(self, local_env: int) -> int:
        return self.first_episode + local_env


SUM_KEYS = ("episodes", "env_steps", "sum_collisions", "sum_qp_infeasible", "sum_return", "sum_return_sq",
            "sum_metric", "sum_success")


def reduce_stats(stats: dict, group=None, device=None) -> dict:
    """All-reduce per-device partial stats: sums, and min of min_pairwise_distance."""
    import torch
    import torch.distributed as dist

    vals = torch.tensor([float(stats[k]) for k in SUM_KEYS], dtype=torch.float64, device=device)
    mn = torch.tensor([float(stats["min_pairwise_distance"])], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(vals, group=group)
        dist.all_reduce(mn, op=dist.ReduceOp.MIN, group=group)
    out = {k: v for k, v in zip(SUM_KEYS, vals.tolist())}
    out["min_pairwise_distance"] = float(mn.item())
    n = max(out["episodes"], 1.0)
    out["mean_return"] = out["sum_return"] / n
    out["success_rate"] = out["sum_success"] / n
    return out
