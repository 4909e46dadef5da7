"""The real multi-process plumbing of row sharding on one B200: two processes
(gloo for the host collectives), each owning half of the rows in a CUDA handle, fold their
`sc_local_red0` vectors, exchange the 64-byte `sc_ipc_handle` blobs and map each other's
mailbox with `sc_connect` (cudaIpcOpenMemHandle), then evaluate the sharded progress
(`sc_progress_parts` + the rank fold).  No persistent kernel is launched: two ranks whose
kernels wait on each other cannot share one GPU (the in-kernel exchange itself is tested
with emulated ranks inside one launch, tests/test_gpu_vworld.py).  The folded values must
equal the single-handle ones."""
import json
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _ys(kind, d, seed):
    rng = np.random.default_rng(seed)
    return [rng.standard_normal(d + (1 if kind == "ses" else 2)) for _ in range(4)]


def _worker(rank, world, port, out_path):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2405_09157_b200 import instances, shard
    comm = shard.Comm()
    res = {}
    inst = instances.gen_ses(5001, 37, 3, "uniform-ball")
    dev = shard.ses_device_sharded(inst, comm)
    assert dev.handle.prob.n_local in (2500, 2501)
    res["ses"] = [dev.progress(y) for y in _ys("ses", inst.d, 1)]
    dev.close()
    sinst, _ = instances.gen_svm(2100, 1900, 29, 4, 1.0)
    dev = shard.svm_device_sharded(sinst, comm)
    res["svm"] = [dev.progress(y) for y in _ys("svm", sinst.d, 2)]
    dev.close()
    if rank == 0:
        with open(out_path, "w") as fh:
            json.dump(res, fh)
    dist.barrier()
    dist.destroy_process_group()


def test_two_process_ipc_connect_and_sharded_progress(tmp_path):
    from paper_2405_09157_b200 import instances, ses, svm
    out = str(tmp_path / "ipc.json")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    got = json.load(open(out))
    inst = instances.gen_ses(5001, 37, 3, "uniform-ball")
    dev = ses.ses_device(inst)
    want = [dev.progress(y) for y in _ys("ses", inst.d, 1)]
    dev.close()
    np.testing.assert_allclose(got["ses"], want, rtol=1e-14, atol=0)
    sinst, _ = instances.gen_svm(2100, 1900, 29, 4, 1.0)
    dev = svm.svm_device(sinst)
    want = [dev.progress(y) for y in _ys("svm", sinst.d, 2)]
    dev.close()
    np.testing.assert_allclose(got["svm"], want, rtol=1e-14, atol=0)
