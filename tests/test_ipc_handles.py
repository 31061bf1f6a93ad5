"""MPMD handle exchange (reference runtime.py:170-233, 390-406):
registry semantics on CPU, and the CUDA-IPC token contract across two real
processes on one GPU (no kernel waits on the other process: the processes
take turns, synchronised through the parent's pipes)."""

import os
import subprocess
import sys

import numpy as np
import pytest

import paper_2601_14466_b200 as bc
from paper_2601_14466_b200 import _lib, ipc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _tok(i):
    return ipc.HandleToken(bytes([i]) * ipc.TOKEN_BYTES, i, 8, "float64", (1,))


def test_registry_publish_collect_rules():
    reg = ipc.HandleRegistry(3, mode="shared_address")
    assert reg.missing == [0, 1, 2] and not reg.complete
    reg.publish(1, "h1")
    with pytest.raises(ipc.RegistryError, match="already published"):
        reg.publish(1, "again")
    with pytest.raises(ipc.RegistryError, match=r"missing devices \[0, 2\]"):
        reg.coordinator_handles()
    with pytest.raises(ValueError):
        reg.publish(3, "x")
    reg.publish(0, "h0")
    reg.publish(2, "h2")
    assert reg.complete and reg.coordinator_handles() == ["h0", "h1", "h2"]
    iso = ipc.HandleRegistry(2)
    iso.publish(0, _tok(1))
    assert iso.missing == [1]


def test_ipc_abi_rejects_null_and_foreign_addresses():
    import ctypes as C

    lib = _lib.load()
    buf = C.create_string_buffer(ipc.TOKEN_BYTES)
    assert lib.bcmg_ipc_export(None, buf) == _lib.BCMG_ERR_CONFIG
    assert lib.bcmg_ipc_open(None, C.byref(C.c_void_p())) == _lib.BCMG_ERR_CONFIG
    assert lib.bcmg_ipc_close_all() == _lib.BCMG_OK


_CHILD = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_2601_14466_b200 import ipc
tok = ipc.HandleToken(bytes.fromhex(sys.stdin.readline().strip()), 0, 8 * 1000, "float64", (10, 100))
t = ipc.open_handle(tok)                      # the parent's tensor, mapped into this process
ok = bool(torch.equal(t.cpu(), torch.arange(1000, dtype=torch.float64).reshape(10, 100)))
t[3:5] *= -2.0                                # write through the mapping
torch.cuda.synchronize()
import ctypes as C
from paper_2601_14466_b200 import _lib
ftok = ipc.HandleToken(bytes.fromhex(sys.stdin.readline().strip()), 0, 16, "int32", (4,))
flag = ipc.open_handle(ftok)                  # the parent's flag words
st = torch.cuda.current_stream()
rc = _lib.load().bcmg_stream_write_flag(C.c_void_p(st.cuda_stream), C.c_void_p(flag.data_ptr() + 4), 7)
st.synchronize()
own = torch.full((7,), 5.0, dtype=torch.float64, device="cuda")
mine = ipc.publish_handle(own, 1)
try:
    ipc.open_handle(mine)                     # a process cannot open its own token
    own_refused = False
except ipc.HandleDomainError:
    own_refused = True
print(int(ok), int(own_refused), mine.token.hex(), rc, flush=True)
sys.stdin.readline()                          # keep `own` alive until the parent has read it
ipc.close_all()
"""


@pytest.mark.gpu
def test_ipc_token_across_processes(cuda):
    import torch

    a = torch.arange(1000, dtype=torch.float64, device=cuda).reshape(10, 100)
    big = torch.empty(1 << 20, dtype=torch.float64, device=cuda)  # an interior address of a larger allocation
    view = big[4096:4096 + 1000].view(10, 100)
    view.copy_(a)
    tok = ipc.publish_handle(view)
    flags = torch.zeros(4, dtype=torch.int32, device=cuda)
    ftok = ipc.publish_handle(flags)
    torch.cuda.synchronize()
    p = subprocess.Popen([sys.executable, "-c", _CHILD, ROOT], stdin=subprocess.PIPE, stdout=subprocess.PIPE,
                         stderr=subprocess.PIPE, text=True)
    try:
        p.stdin.write(tok.token.hex() + "\n" + ftok.token.hex() + "\n")
        p.stdin.flush()
        line = p.stdout.readline().split()
        assert len(line) == 4, p.stderr.read()
        # the child raised flag word 1 with a stream memory operation on the opened token
        # (the copy-engine panel hand-off's flag path, csrc/comm.cpp post_flag)
        assert line[3] == "0", "cuStreamWriteValue32 refused an IPC-mapped address"
        assert flags.cpu().tolist() == [0, 7, 0, 0]
        st = torch.cuda.current_stream()
        lib = _lib.load()
        import ctypes as C

        assert lib.bcmg_stream_wait_flag(C.c_void_p(st.cuda_stream), C.c_void_p(flags.data_ptr() + 4), 7) == 0
        st.synchronize()  # already satisfied: returns
        assert line[0] == "1", "child saw different bytes through the mapping"
        assert line[1] == "1", "opening a process's own token must be refused"
        # the child's writes landed in our memory (the child synchronised before answering)
        want = np.arange(1000, dtype=np.float64).reshape(10, 100)
        want[3:5] *= -2.0
        assert np.array_equal(view.cpu().numpy(), want)
        # the child's own tensor, opened here (the coordinator side of the registry)
        reg = ipc.HandleRegistry(1)
        reg.publish(0, ipc.HandleToken(bytes.fromhex(line[2]), 1, 56, "float64", (7,)))
        (theirs,) = reg.coordinator_handles()
        assert torch.equal(theirs.cpu(), torch.full((7,), 5.0, dtype=torch.float64))
        ipc.close_all()
        p.stdin.write("done\n")
        p.stdin.flush()
        assert p.wait(timeout=120) == 0, p.stderr.read()
    finally:
        if p.poll() is None:
            p.kill()
