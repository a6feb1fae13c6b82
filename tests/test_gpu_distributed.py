"""The pose-sharded product path (distributed.ShardedDRR) at world size 2.

Two ranks share cuda:0 (this run has one GPU) over gloo: the CT is broadcast
from rank 0, each rank walks its block of the global pose batch, and its
kernels store images / loss values / pose gradients straight into rank 0's
buffers through the peer-memory ABI (drr_peer_export / drr_peer_open: CUDA
IPC, the same mechanism that carries the stores over NVLink on a multi-GPU
node) -- or, in the "collective" fallback (peer access unavailable), into
local rows gathered by one collective.  Rank 0's gathered results must equal the single-process batch bit for
bit: the partition has no exchange step, so sharding may not
change any result.  Registration traces of the population study are gathered
in global order and equal single-process traces.
"""

import math
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SP = (2.0, 2.0, 3.0)
TRUTH = (150.0, math.pi / 2, math.pi / 2, 0.0, 0.0, 0.0, 0.0)
N_POSES = 7  # uneven shards: 4 + 3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _inputs():
    from paper_2208_12737_b200 import synthetic
    vol = synthetic.chest_phantom((48, 40, 24))
    poses = synthetic.sample_poses(TRUTH, synthetic.NARROW_HALF_WIDTHS, N_POSES, seed=3)
    return vol, poses


def _worker(rank, world, port, out_dir, peer_mode="peer"):
    import faulthandler
    import traceback
    faulthandler.enable(open(os.path.join(out_dir, f"fault{rank}.txt"), "w"))
    if peer_mode == "collective":
        os.environ["DRR_PEER_MODE"] = "collective"
    try:
        _work(rank, world, port, out_dir)
    except BaseException:
        with open(os.path.join(out_dir, f"error{rank}.txt"), "w") as f:
            f.write(traceback.format_exc())
        raise


def _errors(out_dir):
    msgs = []
    for name in sorted(os.listdir(out_dir)):
        if name.startswith(("error", "fault")):
            text = open(os.path.join(out_dir, name)).read()
            if text.strip():
                msgs.append(f"--- {name}\n{text}")
    return "\n".join(msgs)


def _work(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2208_12737_b200.distributed import ShardedDRR
    from paper_2208_12737_b200.registration import OptimizerConfig
    vol, poses = _inputs()
    sd = ShardedDRR(vol if rank == 0 else None, SP, 150.0, 33, 3.0, width=29,
                    device="cuda:0", ray_split=1)
    want = "collective" if os.environ.get("DRR_PEER_MODE") == "collective" else "peer"
    fixed = sd.render(np.asarray([TRUTH]))
    fixed_all = [fixed.cpu() if rank == 0 else None]
    dist.broadcast_object_list(fixed_all, src=0)
    fixed = fixed_all[0][0].numpy()
    img = sd.render(poses)
    assert all(p.mode == want for p in sd._peer.values()), [p.mode for p in sd._peer.values()]
    img2 = sd.render(poses[::-1].copy())           # buffers reused across calls
    lg = sd.loss_and_gradient(poses, fixed)
    cfg = OptimizerConfig(max_iters=12)
    traces = sd.register_batch(fixed, poses[:5], cfg)
    if rank == 0:
        val, grad = lg
        np.savez(os.path.join(out_dir, "sharded.npz"), img=img.cpu().numpy(),
                 img2=img2.cpu().numpy(), val=val.cpu().numpy(), grad=grad.cpu().numpy(),
                 fixed=fixed, t_losses=np.concatenate([t.losses for t in traces]),
                 t_poses=np.concatenate([t.poses for t in traces]),
                 t_len=np.array([len(t.losses) for t in traces]))
    else:
        assert img is None and lg is None and traces is None
    sd.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("peer_mode", ["peer", "collective"])
def test_two_ranks_match_single_process(cuda_device, tmp_path, peer_mode):
    import torch
    import torch.multiprocessing as mp
    from paper_2208_12737_b200 import DeviceVolume, Detector, pose_frames, render_frames
    from paper_2208_12737_b200.registration import (OptimizerConfig, loss_and_gradient,
                                                    register_batch)
    try:
        mp.spawn(_worker, args=(2, _free_port(), str(tmp_path), peer_mode), nprocs=2, join=True)
    except Exception as exc:
        raise AssertionError(f"{exc}\n{_errors(str(tmp_path))}") from None
    got = dict(np.load(tmp_path / "sharded.npz"))
    vol, poses = _inputs()
    dv = DeviceVolume(vol, SP, device=cuda_device)
    det = Detector(33, 29, 3.0, ray_split=1)
    fr = pose_frames(torch.tensor(poses, device=cuda_device), dv.center).detach()
    img = render_frames(dv, det, fr).cpu().numpy()
    np.testing.assert_array_equal(got["img"], img)
    np.testing.assert_array_equal(got["img2"], img[::-1])
    # the frame from the device pose kernel, as the sharded path makes it (TRUTH's
    # central rays run exactly along a voxel plane, so a 1-ulp different cos(pi/2)
    # from another trig implementation could pick the neighbouring voxel column)
    from paper_2208_12737_b200.renderer import _PoseFrames
    f_truth = _PoseFrames.apply(torch.tensor([TRUTH], dtype=torch.float64, device=cuda_device),
                                dv.center)
    fixed = render_frames(dv, det, f_truth.detach())[0].cpu().numpy()
    np.testing.assert_array_equal(got["fixed"], fixed)
    val, grad = loss_and_gradient(dv, det, torch.tensor(poses, device=cuda_device), fixed)
    np.testing.assert_array_equal(got["val"], val.cpu().numpy())
    np.testing.assert_array_equal(got["grad"], grad.cpu().numpy())
    traces = register_batch(fixed, dv, poses[:5], det, OptimizerConfig(max_iters=12))
    np.testing.assert_array_equal(got["t_len"], [len(t.losses) for t in traces])
    np.testing.assert_array_equal(got["t_losses"], np.concatenate([t.losses for t in traces]))
    np.testing.assert_array_equal(got["t_poses"], np.concatenate([t.poses for t in traces]))


def test_peer_rows_single_process(cuda_device):
    """World of one: PeerRows is a plain local buffer and ShardedDRR is the
    single-GPU path (auto ray split included)."""
    import torch
    from paper_2208_12737_b200 import DeviceVolume, Detector, pose_frames, render_frames
    from paper_2208_12737_b200.distributed import ShardedDRR
    vol, poses = _inputs()
    sd = ShardedDRR(vol, SP, 150.0, 33, 3.0, width=29, device=cuda_device)
    img = sd.render(poses)
    dv = DeviceVolume(vol, SP, device=cuda_device)
    fr = pose_frames(torch.tensor(poses, device=cuda_device), dv.center).detach()
    np.testing.assert_array_equal(img.cpu().numpy(),
                                  render_frames(dv, Detector(33, 29, 3.0), fr).cpu().numpy())
