"""Multi-process host logic of the sensor network on CPU (gloo, world 2):
sensor partitioning and the 360-degree energyscape gather. The per-sensor
energyscape is the C oracle's (the GPU path runs the same gather over NCCL);
the gather's oracle is the concatenation of per-sensor reference images
(SURVEY.md §8(e))."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT, TINY

from paper_2208_10839_b200.distributed import gather_energyscapes, sensor_serial, sensors_for_rank, view_360


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _sensor_image(sensor, trigger_seq=0):
    import sys
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as po
    port = po.Port()
    mics = port.default_array(42)
    cfg = po.Config(mic_xyz=mics, directions=port.direction_grid(0), **TINY)
    serial = sensor_serial(sensor)
    # per-sensor scene: one reflector whose azimuth depends on the sensor
    pk = port.synthesize(cfg, [(1.0, -0.6 + 0.3 * sensor, 0.0, 0.5)], 0.01,
                         7 + 1000 * serial + trigger_seq)
    return port.process(cfg, pk)


def _worker(rank, world, port_no, n_sensors, result_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = sensors_for_rank(n_sensors, world, rank)
    local = torch.from_numpy(np.stack([_sensor_image(s) for s in mine]))
    g = gather_energyscapes(local, dst=0)
    if rank == 0:
        v = view_360(g, n_sensors)
        np.save(result_path, v.numpy())
    else:
        assert g is None
    dist.barrier()
    dist.destroy_process_group()


def test_sensors_for_rank_partition():
    for world in (1, 2, 4, 8):
        owned = [sensors_for_rank(8, world, r) for r in range(world)]
        flat = sorted(s for o in owned for s in o)
        assert flat == list(range(8))
        assert all(len(o) == 8 // world for o in owned)
    assert [sensor_serial(s) for s in range(8)] == list(range(1, 9))


@pytest.mark.parametrize("n_sensors", [2, 4])
def test_gather_360_world2_gloo(tmp_path, n_sensors):
    out = str(tmp_path / "view.npy")
    mp.spawn(_worker, args=(2, _free_port(), n_sensors, out), nprocs=2, join=True)
    view = np.load(out)
    want = np.stack([_sensor_image(s) for s in range(n_sensors)])
    assert view.shape == want.shape == (n_sensors, 90, 58)
    assert np.array_equal(view, want)
    # each sensor's reflector lands at a different azimuth cell
    peaks = [np.unravel_index(np.argmax(v), v.shape)[0] for v in view]
    assert len(set(peaks)) == n_sensors
