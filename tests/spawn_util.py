"""Multi-process test launcher: one spawned process per rank, results over a
queue.  A rendezvous port taken between the probe and the bind (EADDRINUSE)
makes the workers report "__init_failed__ ..." instead of raising; the ranks
are then stopped and the run repeated on a new port (up to `attempts`)."""
import queue
import socket


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def init_failed(rank, q, exc):
    """For a worker's init_process_group failure: report it (no raise)."""
    q.put((rank, f"__init_failed__ {exc!r}"))


def spawn_ranks(world, make_args, target, timeout, attempts=3):
    """Run target(*make_args(rank, port, q)) on `world` spawned processes;
    returns {rank: result}."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    res = {}
    for attempt in range(attempts):
        q = ctx.Queue()
        port = free_port()
        procs = [ctx.Process(target=target, args=make_args(r, port, q)) for r in range(world)]
        for p in procs:
            p.start()
        res = {}
        retry = False
        try:
            while len(res) < world:
                r, v = q.get(timeout=timeout)
                res[r] = v
                if isinstance(v, str) and v.startswith("__init_failed__"):
                    retry = True
                    break
        except queue.Empty:
            pass
        if retry:
            for p in procs:
                p.terminate()
        for p in procs:
            p.join(timeout=60)
        if not retry or attempt == attempts - 1:
            return res
    return res
