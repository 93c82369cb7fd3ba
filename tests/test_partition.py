"""Multi-rank slab protocol (the P-way generalisation of the reference's
run_heterogeneous) on world_size 2 and 3 with gloo + CPU tensors.  The step
engine here is the oracle (tests may use it); on GPUs the same SlabRunner
drives tsr_advance and exchanges over NCCL."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, name, extent, steps, k, poison, out_dir, overlap=False):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    import oracle
    import paper_2303_08365_b200 as ts
    from paper_2303_08365_b200.partition import SlabRunner, local_from_global, plan_slabs
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = oracle.Oracle()
    kern = ts.find_benchmark(name).kernel
    glob = ts.Grid(extent, [kern.radius] * len(extent))
    orc.fill_random(glob, 500)
    plan = plan_slabs(extent, kern.radius, k, world, rank)
    loc = local_from_global(glob, plan, poison=poison)
    runner = SlabRunner.on_host(plan, loc, lambda g, n: orc.naive_run(g, kern, n),
                                overlap=overlap)
    runner.run(steps)
    np.save(os.path.join(out_dir, f"own{rank}.npy"), runner.own_rows())
    np.save(os.path.join(out_dir, f"log{rank}.npy"),
            np.array([len(runner.log.records), runner.round, runner.log.ghost_recompute_points]))
    dist.barrier()
    dist.destroy_process_group()


def _run(tmp_path, world, name, extent, steps, k, poison=True, overlap=False):
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, name, extent, steps, k, poison,
                                      str(tmp_path), overlap), nprocs=world, join=True,
                       start_method="spawn")
    return ([np.load(tmp_path / f"own{r}.npy") for r in range(world)],
            [np.load(tmp_path / f"log{r}.npy") for r in range(world)])


@pytest.mark.parametrize("overlap", [False, True], ids=["serial", "overlap"])
@pytest.mark.parametrize("world,name,extent,steps,k", [
    (2, "Heat-2D", [128, 64], 6, 3),      # test_scheduler.cpp:137-158's shape
    (2, "Box-2D9P", [80, 24], 5, 2),
    (3, "Heat-2D", [61, 37], 7, 3),
    (3, "Heat-3D", [30, 9, 11], 5, 2),
    (2, "Star-2D9P", [48, 20], 6, 4),
    (3, "Heat-2D", [13, 20], 5, 2),      # slabs of 4-5 planes: no interior range
])
def test_slabs_equal_oracle_bitwise(ts, orc, tmp_path, world, name, extent, steps, k, overlap):
    """Serial rounds (exchange, then the whole slab) and overlapped rounds
    (interior range, exchange, seam ranges) are both bitwise naive_run."""
    own, logs = _run(tmp_path, world, name, extent, steps, k, overlap=overlap)
    kern = ts.find_benchmark(name).kernel
    ref = ts.Grid(extent, [kern.radius] * len(extent))
    orc.fill_random(ref, 500)
    orc.naive_run(ref, kern, steps)
    h = kern.radius
    got = np.concatenate(own, axis=0)
    want = ref.padded(ref.parity)[h:h + extent[0]]
    assert np.isfinite(got).all()  # NaN-poisoned seam halos never reached owned rows
    assert got.tobytes() == want.tobytes()
    rounds = -(-steps // k)
    # one message per direction per seam per round (2*ceil(T/tb) for 2 workers)
    assert sum(int(l[0]) for l in logs) == 2 * (world - 1) * rounds
    assert all(int(l[1]) == rounds for l in logs)


def test_reference_message_and_ghost_counts(ts, orc, tmp_path):
    """test_scheduler.cpp:137-158: T=6, tb=3 on 128x64 -> 4 messages of
    3*64*8 bytes; our ghost recompute counts full ghost slabs per step."""
    from paper_2303_08365_b200.partition import plan_slabs
    p0 = plan_slabs([128, 64], 1, 3, 2, 0)
    p1 = plan_slabs([128, 64], 1, 3, 2, 1)
    assert (p0.own_lo, p0.own_hi, p1.own_lo, p1.own_hi) == (0, 64, 64, 128)
    assert p0.depth == 3 and p0.bytes_per_message == 3 * 64 * 8
    assert p0.local_extent == [67, 64] and p1.local_extent == [67, 64]
    with pytest.raises(ValueError):
        plan_slabs([8, 8], 1, 5, 2, 0)  # subdomain smaller than the halo depth


def _gpu_worker(rank, world, port, name, extent, steps, k, out_dir, mode):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    import oracle
    import paper_2303_08365_b200 as ts
    from paper_2303_08365_b200.partition import SlabRunner, local_from_global, plan_slabs
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    orc = oracle.Oracle()
    kern = ts.find_benchmark(name).kernel
    glob = ts.Grid(extent, [kern.radius] * len(extent))
    orc.fill_random(glob, 500)
    plan = plan_slabs(extent, kern.radius, k, world, rank)
    loc = local_from_global(glob, plan, poison=True)
    runner = SlabRunner.on_device(ts, kern, plan, loc, torch.device("cuda", 0),
                                  overlap=mode != "serial",
                                  transport="peer" if mode.startswith("peer") else "nccl",
                                  graphs=mode == "peer_graph")
    runner.run(steps)
    runner.close()  # peer transport: every neighbour's stores have landed
    np.save(os.path.join(out_dir, f"own{rank}.npy"), runner.own_rows(loc))
    np.save(os.path.join(out_dir, f"log{rank}.npy"),
            np.array([len(runner.log.records), runner.round, runner.log.ghost_recompute_points]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["serial", "overlap", "peer", "peer_graph"])
@pytest.mark.parametrize("world,name,extent,steps,k", [
    (2, "Heat-3D", [70, 40, 67], 7, 3),   # tb3d engine on each slab
    (3, "Box-2D9P", [90, 130], 9, 4),    # stream2d engine
    (2, "Box-3D27P", [40, 30, 50], 4, 1),  # box3d engine
    (2, "Box-3D27P", [44, 30, 50], 5, 2),  # box3d two-level engine
    (3, "Heat-1D", [300], 7, 3),          # stream1d engine, 1-D slabs
])
def test_slabs_on_device_equal_oracle(ts, orc, tmp_path, world, name, extent, steps, k, mode):
    """The device slab state (pitched HBM buffers, tsr_advance or
    tsr_sweep_range on two streams, zero-copy plane views) with several ranks
    sharing one GPU over gloo; `peer`: the seam passes store straight into the
    neighbour processes' ghost planes through CUDA IPC mappings and the
    rounds are ordered by device-side flags (no message on the data path);
    `peer_graph`: after the first full round every full round is a replayed
    CUDA graph (one per buffer parity; a few more rounds so both replay)."""
    if mode == "peer_graph":
        steps += 3 * k
    port = _free_port()
    mp.start_processes(_gpu_worker, args=(world, port, name, extent, steps, k, str(tmp_path),
                                          mode),
                       nprocs=world, join=True, start_method="spawn")
    kern = ts.find_benchmark(name).kernel
    ref = ts.Grid(extent, [kern.radius] * len(extent))
    orc.fill_random(ref, 500)
    orc.naive_run(ref, kern, steps)
    h = kern.radius
    got = np.concatenate([np.load(tmp_path / f"own{r}.npy") for r in range(world)], axis=0)
    want = ref.padded(ref.parity)[h:h + extent[0]]
    assert np.isfinite(got).all()
    assert got.tobytes() == want.tobytes()


@pytest.mark.parametrize("world,n0,radius,k", [(2, 128, 1, 3), (3, 61, 1, 2), (4, 40, 2, 2),
                                               (8, 1024, 1, 3), (5, 23, 1, 4)])
def test_peer_mirror_shift_lands_on_neighbour_ghosts(world, n0, radius, k):
    """The plane shift PeerLink gives each seam pass maps the sender's
    boundary own planes exactly onto the receiver's ghost planes, in the
    receiver's local coordinates (so a round's seam passes deliver the same
    planes the NCCL transport sends)."""
    from paper_2303_08365_b200.partition import mirror_shift, plan_slabs
    plans = [plan_slabs([n0, 7], radius, k, world, r) for r in range(world)]
    for r, p in enumerate(plans):
        g = lambda plan, local: local - plan.ghost_lo + plan.own_lo  # local row -> global row
        if r > 0:  # lo seam: my first depth own planes -> lo neighbour's ghost_hi planes
            nb = plans[r - 1]
            shift = mirror_shift(p, "lo")
            for j in range(p.depth):
                mine = p.ghost_lo + j
                theirs = mine + shift
                assert nb.ghost_lo + nb.own <= theirs < nb.local_extent[0]
                assert g(p, mine) == g(nb, theirs)
        if r < world - 1:  # hi seam: my last depth own planes -> hi neighbour's ghost_lo
            nb = plans[r + 1]
            shift = mirror_shift(p, "hi")
            for j in range(p.depth):
                mine = p.ghost_lo + p.own - p.depth + j
                theirs = mine + shift
                assert 0 <= theirs < nb.ghost_lo
                assert g(p, mine) == g(nb, theirs)
