"""Multi-rank pipeline transport logic on CPU (gloo, world size 2 and 4).

The device trainer (csrc/device/trainer.cpp, Trainer::step) drives P2P with four
communicators: activations r->r+1 on comm_act[r % 2], gradients r->r-1 on
comm_grad[r % 2], each on its own stream, compute waiting on receive events and
send streams waiting on compute. This test replays exactly that issue program
(same rank action lists from libpf_host's build_schedule, same channel/peer
rules) with one thread per stream and gloo process groups standing in for the
NCCL communicators, and checks that it completes (no deadlock) and that every
stage consumes the payload of the right (microbatch, stage) edge of the DAG
(rule 3, proj/src/dag.cpp:90-93).
"""
import os
import queue
import threading

import pytest


def _worker(rank, world, kind, M, port, errq):
    import torch
    import torch.distributed as dist

    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        groups = {name: dist.new_group(list(range(world)), backend="gloo")
                  for name in ("act0", "act1", "grad0", "grad1")}
        from paper_2602_05754_b200 import pipefreeze as pf

        cfg = pf.PipelineConfig(kind, world, 1, M)
        actions = pf.build_schedule(cfg).rank_order[rank]
        S = world
        stage = rank + 1

        class Stream:
            """In-order op queue on a thread (a CUDA stream stand-in)."""

            def __init__(self):
                self.q = queue.Queue()
                self.t = threading.Thread(target=self.run, daemon=True)
                self.t.start()

            def run(self):
                while True:
                    fn = self.q.get()
                    if fn is None:
                        return
                    fn()

            def submit(self, fn):
                done = threading.Event()

                def op():
                    fn()
                    done.set()

                self.q.put(op)
                return done

            def close(self):
                self.q.put(None)
                self.t.join(timeout=60)

        act_send, act_recv, grad_send, grad_recv = Stream(), Stream(), Stream(), Stream()
        consumed = []
        pending_sends = []
        for a in actions:
            m = a.microbatch
            if a.kind == 0:  # forward f(m, s)
                if stage > 1:
                    buf = torch.zeros(2)
                    ev = act_recv.submit(lambda b=buf: dist.recv(b, src=rank - 1, group=groups[f"act{(rank - 1) % 2}"]))
                    assert ev.wait(60), "activation receive timed out"
                    assert buf.tolist() == [m, stage - 1], (buf.tolist(), m, stage)
                    consumed.append(("f", m))
                out = torch.tensor([float(m), float(stage)])
                if stage < S:
                    pending_sends.append(act_send.submit(
                        lambda t=out: dist.send(t, dst=rank + 1, group=groups[f"act{rank % 2}"])))
            else:  # backward b(m, s)
                if stage < S:
                    buf = torch.zeros(2)
                    ev = grad_recv.submit(lambda b=buf: dist.recv(b, src=rank + 1, group=groups[f"grad{(rank + 1) % 2}"]))
                    assert ev.wait(60), "gradient receive timed out"
                    assert buf.tolist() == [-m, stage + 1], (buf.tolist(), m, stage)
                    consumed.append(("b", m))
                g = torch.tensor([-float(m), float(stage)])
                if stage > 1:
                    pending_sends.append(grad_send.submit(
                        lambda t=g: dist.send(t, dst=rank - 1, group=groups[f"grad{rank % 2}"])))
        for ev in pending_sends:
            assert ev.wait(60), "send never matched"
        for s in (act_send, act_recv, grad_send, grad_recv):
            s.close()
        # every remote input of this stage arrived exactly once, in schedule order
        exp = [("f", a.microbatch) for a in actions if a.kind == 0 and stage > 1] + \
              [("b", a.microbatch) for a in actions if a.kind == 1 and stage < S]
        assert sorted(consumed) == sorted(exp)
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback

        errq.put(f"rank {rank}: {e!r}\n{traceback.format_exc()}")


@pytest.mark.parametrize("kind,world,M", [("1f1b", 2, 4), ("gpipe", 2, 3), ("1f1b", 4, 8), ("gpipe", 4, 2)])
def test_p2p_issue_program_completes_and_routes(kind, world, M):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    errq = ctx.Queue()
    port = 29500 + hash((kind, world, M)) % 1000
    procs = [ctx.Process(target=_worker, args=(r, world, kind, M, port, errq)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not errs, "\n".join(errs)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
