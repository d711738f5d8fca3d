"""world_size-2 gloo tests (CPU) of the multi-GPU host logic: band/view partitioning and the final
gather, with the device renderer replaced by a deterministic per-pixel function."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2206_10885_b200 import dist as kd


def test_shard_rows_tiles_the_frame():
    for h, w in [(1080, 8), (7, 3), (2, 4), (1, 2), (100, 1)]:
        bands = [kd.shard_rows(h, r, w) for r in range(w)]
        assert bands[0][0] == 0 and bands[-1][1] == h
        assert all(a[1] == b[0] for a, b in zip(bands, bands[1:]))
        sizes = [b[1] - b[0] for b in bands]
        assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        kd.shard_rows(10, 2, 2)


def test_shard_views_round_robin():
    assert kd.shard_views(10, 1, 4) == [1, 5, 9]
    seen = sorted(v for r in range(3) for v in kd.shard_views(100, r, 3))
    assert seen == list(range(100))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _fake_bands(width):
    def render_rows(r0, r1):
        rows = torch.arange(r0, r1, dtype=torch.float32)[:, None]
        cols = torch.arange(width, dtype=torch.float32)[None, :]
        color = torch.stack([rows + 0 * cols, 0 * rows + cols, rows * cols], dim=2)
        depth = rows * 1000 + cols
        return color, depth, -color, ((rows + cols) % 2).to(torch.uint8)

    return render_rows


def test_interleaved_bands_tile_the_frame():
    for h, w, band in [(1080, 8, 32), (1080, 3, 32), (7, 2, 2), (5, 4, 32), (33, 2, 8)]:
        owned = np.full(h, -1)
        for r in range(w):
            for r0, r1 in kd.shard_rows_interleaved(h, r, w, band):
                assert np.all(owned[r0:r1] == -1) and r1 - r0 <= band
                owned[r0:r1] = r
        assert np.all(owned >= 0)
        rows = [int((owned == r).sum()) for r in range(w)]
        assert max(rows) - min(rows) <= band  # balanced to within one band
    with pytest.raises(ValueError):
        kd.shard_rows_interleaved(10, 0, 2, 0)


def _worker(rank, world, port, height, width, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        class Pose:
            pass

        pose = Pose()
        pose.height, pose.width = height, width
        color, depth, normal, hit = kd.render_frame_sharded(None, pose, settings=object(), render_rows=_fake_bands(width))
        views = kd.gather_views(torch.full((2, 3), float(rank)))
        inter = kd.render_frame_sharded(None, pose, settings=object(), render_rows=_fake_bands(width), interleave=2)
        hdr = kd.render_pathtraced_sharded(None, pose, spp=1, seed=0, interleave=3,
                                           pathtrace_rows=lambda r0, r1: _fake_bands(width)(r0, r1)[0].double())
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), color=color.numpy(), depth=depth.numpy(), normal=normal.numpy(),
                 hit=hit.numpy(), views=views.numpy(), icolor=inter[0].numpy(), idepth=inter[1].numpy(), inormal=inter[2].numpy(),
                 ihit=inter[3].numpy(), hdr=hdr.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("height", [9, 1])
def test_sharded_frame_equals_single_process(tmp_path, height):
    world, width = 2, 5
    mp.spawn(_worker, args=(world, _free_port(), height, width, str(tmp_path)), nprocs=world, join=True)
    want = _fake_bands(width)(0, height)
    for r in range(world):
        got = np.load(tmp_path / f"r{r}.npz")
        assert np.array_equal(got["color"], want[0].numpy())
        assert np.array_equal(got["depth"], want[1].numpy())
        assert np.array_equal(got["normal"], want[2].numpy())
        assert np.array_equal(got["hit"], want[3].numpy())
        assert np.array_equal(got["views"][:, 0, 0], np.arange(world, dtype=np.float32))
        # bands of 2 rows dealt round-robin, reassembled in image order
        assert np.array_equal(got["icolor"], want[0].numpy()) and np.array_equal(got["idepth"], want[1].numpy())
        assert np.array_equal(got["inormal"], want[2].numpy()) and np.array_equal(got["ihit"], want[3].numpy())
        assert np.array_equal(got["hdr"], want[0].double().numpy())  # path-traced bands of 3 rows
