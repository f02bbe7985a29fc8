"""Multi-rank pipeline transport logic on CPU (gloo, world size 2 and 4).

The device trainer (csrc/device/trainer.cpp, Trainer::step) drives P2P over one two-rank
communicator and stream per link: a cross-rank (activation | gradient, src rank, dst rank)
class of DAG rule-3 edges (pipefreeze.p2p_links). Compute waits on receive events; sends
wait on compute; neighbouring stages on the same rank hand over locally. This test replays
the product's own issue program (pipefreeze.issue_program = libpf_host issue_program, the
list Trainer::step walks), with the same link rules, over every placement: gpipe / 1f1b chains, the interleaved ring, the ZBV V with
activations flowing both ways, zbv-split's W actions) with one thread per link stream and a
gloo process group per link standing in for the NCCL communicators, and checks that it
completes (no deadlock) and that every stage consumes the payload of the right
(microbatch, stage) edge of the DAG (rule 3, proj/src/dag.cpp:90-93).
"""
import os
import queue
import threading

import pytest


def _worker(rank, world, kind, C, M, port, errq):
    import torch
    import torch.distributed as dist

    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2602_05754_b200 import pipefreeze as pf

        cfg = pf.PipelineConfig(kind, world, C, M)
        links = pf.p2p_links(cfg)
        groups = {l: dist.new_group([l[1], l[2]], backend="gloo") for l in links}  # collective, same order
        actions = pf.build_schedule(cfg).rank_order[rank]
        S = cfg.total_stages
        rank_of = {s: pf.stage_to_rank(cfg, s) for s in range(1, S + 1)}

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

        streams = {l: Stream() for l in links if rank in (l[1], l[2])}
        consumed = []
        pending_sends = []
        # the product's issue program (libpf_host issue_program, the list trainer.cpp walks)
        for a, recv_from, send_to in pf.issue_program(cfg, rank):
            m, s = a.microbatch, a.stage
            if a.kind == 2:
                assert recv_from == -1 and send_to == -1  # w(m, s): local dW only
                continue
            edge = a.kind  # 0: activations of f, 1: gradients of b
            if recv_from >= 0:
                l = (edge, recv_from, rank)
                buf = torch.zeros(2)
                ev = streams[l].submit(lambda b=buf, l=l: dist.recv(b, src=l[1], group=groups[l]))
                assert ev.wait(60), f"receive timed out at {a}"
                want = [m, s - 1] if edge == 0 else [-m, s + 1]
                assert buf.tolist() == want, (buf.tolist(), a)
                consumed.append(("fb"[edge], m, s))
            if send_to >= 0:
                l = (edge, rank, send_to)
                out = torch.tensor([float(m), float(s)]) if edge == 0 else torch.tensor([-float(m), float(s)])
                pending_sends.append(streams[l].submit(lambda t=out, l=l: dist.send(t, dst=l[2], group=groups[l])))
        for ev in pending_sends:
            assert ev.wait(60), "send never matched"
        for st in streams.values():
            st.close()
        # every remote input of this rank's stages arrived exactly once
        exp = [("f", a.microbatch, a.stage) for a in actions
               if a.kind == 0 and a.stage > 1 and rank_of[a.stage - 1] != rank] + \
              [("b", a.microbatch, a.stage) for a in actions
               if a.kind == 1 and a.stage < S and rank_of[a.stage + 1] != rank]
        assert sorted(consumed) == sorted(exp)
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback

        errq.put(f"rank {rank}: {e!r}\n{traceback.format_exc()}")


@pytest.mark.parametrize("kind,world,C,M", [("1f1b", 2, 1, 4), ("gpipe", 2, 1, 3), ("1f1b", 4, 1, 8), ("gpipe", 4, 1, 2),
                                            ("interleaved-1f1b", 2, 2, 4), ("interleaved-1f1b", 4, 2, 8),
                                            ("zbv", 2, 2, 4), ("zbv", 4, 2, 8), ("zbv-split", 2, 2, 4),
                                            ("zbv-split", 4, 2, 6)])
def test_p2p_issue_program_completes_and_routes(kind, world, C, M):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    errq = ctx.Queue()
    port = 29500 + (abs(hash((kind, world, C, M))) % 2000)
    procs = [ctx.Process(target=_worker, args=(r, world, kind, C, M, port, errq)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not errs, "\n".join(errs)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]


@pytest.mark.parametrize("kind,world,C", [("1f1b", 4, 1), ("interleaved-1f1b", 4, 2), ("zbv", 4, 2)])
def test_p2p_links_cover_every_cross_rank_edge(kind, world, C):
    from paper_2602_05754_b200 import pipefreeze as pf

    cfg = pf.PipelineConfig(kind, world, C, 4)
    links = pf.p2p_links(cfg)
    S = cfg.total_stages
    for s in range(1, S):
        a, b = pf.stage_to_rank(cfg, s), pf.stage_to_rank(cfg, s + 1)
        if a != b:
            assert (0, a, b) in links and (1, b, a) in links
    assert len(set(links)) == len(links)
    if kind == "interleaved-1f1b":
        assert (0, world - 1, 0) in links  # the ring's wrap-around edge
    if kind == "zbv":
        assert (0, 1, 0) in links and (0, 0, 1) in links  # the V: activations both ways
