"""Multi-GPU layout of the sensor network (one process per GPU).

The reference scales by giving every worker its own Workspace with no shared
state (central_node.cpp:48-53): measurements and sensors are
independent. Here sensor s is processed by rank s mod world; the data path
has no collective. The only exchange is the multi-sensor 360-degree view: the
energyscapes of one trigger (all sensors share (timestamp_us, seq),
sync.hpp:16-19) are gathered to a root rank. Its oracle is the concatenation
of the per-sensor reference images, sensor-major.

Two transports with the same layout (rank-major (world, S_local, n_dirs,
bins), then `view_360` into sensor order):
  * `ViewGather` — the product path on GPUs: the C++ NCCL gather behind the
    C ABI (sn_gather_*, csrc/gather.cpp) on its own stream, double-buffered,
    with the trigger ids checked on the root;
  * `gather_energyscapes` — torch.distributed (gloo in the CPU tests of the
    host logic).
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional, Sequence, Tuple

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
    """Gather equally-shaped per-rank energyscape batches to `dst` over
    torch.distributed. local: (S_local, n_dirs, bins) float32. Returns on
    `dst` a (world, S_local, n_dirs, bins) tensor in rank order, None elsewhere."""
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


def triggers_synchronized(ids: Sequence[Tuple[int, int, int]], world: int) -> bool:
    """Rank-major (serial, timestamp_us, seq) ids of one gather: every rank's
    image i carries the same (timestamp_us, seq) (sync.hpp:16-19)."""
    c = len(ids) // world
    return all(ids[r * c + i][1:] == ids[i][1:] for r in range(world) for i in range(c))


class ViewGather:
    """The C++ NCCL 360-degree gather (sn_gather_*) of one rank.

        g = ViewGather(image_floats=n_dirs * bins, max_count=S_local)   # collective
        g.wait(slot, stream)                    # before overwriting slot's images
        ... process into images[slot] on `stream` ...
        g.start(slot, images[slot], ids, view[slot] (rank 0), stream)
        g.ids(slot) -> ([(serial, ts, seq)], synchronized)   # rank 0

    The NCCL unique id travels over the default torch.distributed group.
    """

    def __init__(self, image_floats: int, max_count: int, device: Optional[int] = None,
                 group: Optional[dist.ProcessGroup] = None):
        import paper_2208_10839_b200 as sn
        self._sn = sn
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.device = torch.cuda.current_device() if device is None else int(device)
        uid = (C.c_uint8 * 128)()
        if self.rank == 0:
            sn._check(sn.lib().sn_gather_unique_id(uid))
        box = [bytes(uid)]
        dist.broadcast_object_list(box, src=0, group=group)
        uid = (C.c_uint8 * 128).from_buffer_copy(box[0])
        h = C.c_void_p()
        sn._check(sn.lib().sn_gather_create(self.rank, self.world, uid, self.device, int(image_floats),
                                            int(max_count), C.byref(h)))
        self._h = h
        self.max_count = int(max_count)
        self._count = [0, 0]

    def start(self, slot: int, images_ptr: int, ids: Sequence[Tuple[int, int, int]], view_ptr: int = 0,
              stream: int = 0):
        n = len(ids)
        self._count[slot] = n
        arr = (self._sn.FrameId * n)(*[self._sn.FrameId(s, 0, t, q) for s, t, q in ids])
        self._sn._check(self._sn.lib().sn_gather_start(self._h, slot, C.c_void_p(images_ptr), arr, n,
                                                       C.c_void_p(view_ptr or None), C.c_void_p(stream or 1)))

    def wait(self, slot: int, stream: Optional[int] = None):
        self._sn._check(self._sn.lib().sn_gather_wait(self._h, slot, C.c_void_p(stream) if stream else None))

    def ids(self, slot: int):
        n = self.world * self._count[slot]
        arr = (self._sn.FrameId * max(1, n))()
        ok = C.c_int32(0)
        self._sn._check(self._sn.lib().sn_gather_ids(self._h, slot, arr, n, C.byref(ok)))
        return [(a.sensor_serial, a.timestamp_us, a.seq) for a in arr[:n]], bool(ok.value)

    def elapsed_ms(self, slot: int) -> float:
        v = C.c_float(0)
        self._sn._check(self._sn.lib().sn_gather_elapsed(self._h, slot, C.byref(v)))
        return float(v.value)

    def close(self):
        if getattr(self, "_h", None):
            self._sn.lib().sn_gather_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
