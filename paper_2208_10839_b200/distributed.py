"""Multi-GPU layout of the sensor network (one process per GPU).

The reference scales by giving every worker its own Workspace with no shared
state (central_node.cpp:48-53): measurements and sensors are
independent. Here sensor s is processed by rank s mod world; the data path
has no collective. The only exchange is the multi-sensor 360-degree view: the
energyscapes of one trigger (all sensors share (timestamp_us, seq),
sync.hpp:16-19) are gathered to a root rank over NCCL (NVLink/NVSwitch). Its
oracle is the concatenation of the per-sensor reference images, sensor-major
(SURVEY.md §8(e)).

Works with any torch.distributed backend ("nccl" on GPUs, "gloo" in the CPU
tests).
"""
from __future__ import annotations

from typing import List, Optional

import torch
import torch.distributed as dist


def sensors_for_rank(n_sensors: int, world: int, rank: int) -> List[int]:
    """Sensor indices (0-based) owned by `rank`: s mod world == rank."""
    return [s for s in range(n_sensors) if s % world == rank]


def sensor_serial(sensor_index: int) -> int:
    """Serial numbers start at 1 (serials 1..8)."""
    return sensor_index + 1


def gather_energyscapes(local: torch.Tensor, dst: int = 0,
                        group: Optional[dist.ProcessGroup] = None) -> Optional[torch.Tensor]:
    """Gather equally-shaped per-rank energyscape batches to `dst`.

    local: (S_local, n_dirs, bins) float32 on this rank's device (NCCL) or CPU
    (gloo). Returns on `dst` a (world, S_local, n_dirs, bins) tensor in rank
    order, None elsewhere.
    """
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if world == 1:
        return local.unsqueeze(0)
    if rank == dst:
        bufs = [torch.empty_like(local) for _ in range(world)]
        dist.gather(local.contiguous(), bufs, dst=dst, group=group)
        return torch.stack(bufs)
    dist.gather(local.contiguous(), None, dst=dst, group=group)
    return None


def view_360(gathered: torch.Tensor, n_sensors: int) -> torch.Tensor:
    """Reorder a (world, S_local, n_dirs, bins) gather into sensor order
    (n_sensors, n_dirs, bins): sensor s sits at [s mod world, s // world]."""
    world = gathered.shape[0]
    out = [gathered[s % world, s // world] for s in range(n_sensors)]
    return torch.stack(out)
