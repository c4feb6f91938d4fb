"""bench.py's multi-rank code path on the one GPU of the test box:
launched by torchrun at world size 1 it initialises the NCCL process group, installs the
bucketed all-reduce as the library's gradient-ready hook (dist.BucketAllReduce), captures
the step (kernels + NCCL all-reduces) in a CUDA graph, and prints one JSON line."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import mpf_synth as S

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("workload,exchange", [("cfg2", "nccl"), ("cfg5", "nccl"), ("cfg2", "peer"), ("cfg5", "peer")])
def test_torchrun_world1_nccl_path(workload, exchange):
    """Both gradient exchanges of the multi-rank path: peer memory (dist.PeerExchange: CUDA IPC
    export, handle all-gather, pushes in the backward, sum in the SGD kernel; the default) and
    the bucketed NCCL all-reduce."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "1",
           "--steps", "3", "--warmup", "3", "--workload", workload, "--no-cpu-baseline", "--exchange", exchange]
    env = dict(os.environ, NCCL_DEBUG="WARN")
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    line = json.loads(lines[0])
    print(workload, "torchrun world 1:", {k: line[k] for k in ("value", "ms_per_step", "gpu_launches")},
          line["config"].get("cuda_graph"), r.stderr[-500:])
    assert line["n_gpus"] == 1 and line["config"]["parallelism"] == "dp1" and line["value"] > 0
    assert line["config"]["grad_exchange"] == exchange
    assert line["e2e"]["value"] > 0


def test_grad_hook_reports_the_bucket_plan():
    """mpf_net_set_grad_hook: one call per conv/FC layer, top down, with the buckets of
    dist.grad_buckets (they tile the gradient buffer), on a CUDA stream; and the gradients
    are those of a step without the hook, bitwise."""
    from paper_1302_1690_b200 import dist as D
    from paper_1302_1690_b200.net import MPFNet
    cfg = S.CONFIGS["cfg2"]
    images, labels = S.make_batch(cfg, [0, 1])
    params = S.init_params(cfg).astype(np.float32)
    img, lab = torch.tensor(images, device="cuda"), torch.tensor(labels, device="cuda")
    net = MPFNet(cfg.layers, cfg.P, cfg.H, cfg.W, max_images=2)
    net.set_params(params)
    net.train_step(img, lab)
    ref = net.grads.clone()
    calls = []
    net.set_grad_hook(lambda l, o, c, s: calls.append((l, o, c, s)))
    net.zero_grads()
    net.train_step(img, lab)
    torch.cuda.synchronize()
    assert [c[:3] for c in calls] == D.grad_buckets(cfg.layers, net.geom.w_offset, net.geom.n_params)
    assert all(c[3] for c in calls)
    assert torch.equal(net.grads, ref)
    net.set_grad_hook(None)
    calls.clear()
    net.train_step(img, lab)
    assert calls == []
