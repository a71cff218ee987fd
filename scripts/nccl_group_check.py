"""Does this image's NCCL accept a collective and point-to-point calls in ONE
group (what comm_iter_exchange issues every CG iteration at N > 1)?  One
rank, one GPU: AllGather + Send/Recv to self inside ncclGroupStart/End, then
checks the data.  Prints one JSON line.
    python scripts/nccl_group_check.py
"""
import ctypes as C
import json

import torch


class UniqueId(C.Structure):
    _fields_ = [("internal", C.c_char * 128)]


def main():
    torch.cuda.init()
    torch.empty(1, device="cuda")  # context
    lib = C.CDLL("libnccl.so.2", mode=C.RTLD_GLOBAL)
    ver = C.c_int()
    lib.ncclGetVersion(C.byref(ver))
    uid = UniqueId()
    assert lib.ncclGetUniqueId(C.byref(uid)) == 0
    comm = C.c_void_p()
    assert lib.ncclCommInitRank(C.byref(comm), 1, uid, 0) == 0
    st = torch.cuda.current_stream().cuda_stream
    send = torch.arange(8, dtype=torch.float64, device="cuda")
    gath = torch.zeros(8, dtype=torch.float64, device="cuda")
    rows = torch.arange(4096, dtype=torch.float64, device="cuda") + 1.0
    recv = torch.zeros_like(rows)
    NCCL_FLOAT64 = 8
    rc = [lib.ncclGroupStart()]
    rc.append(lib.ncclAllGather(C.c_void_p(send.data_ptr()), C.c_void_p(gath.data_ptr()),
                                C.c_size_t(8), NCCL_FLOAT64, comm, C.c_void_p(st)))
    rc.append(lib.ncclSend(C.c_void_p(rows.data_ptr()), C.c_size_t(4096), NCCL_FLOAT64, 0, comm,
                           C.c_void_p(st)))
    rc.append(lib.ncclRecv(C.c_void_p(recv.data_ptr()), C.c_size_t(4096), NCCL_FLOAT64, 0, comm,
                           C.c_void_p(st)))
    rc.append(lib.ncclGroupEnd())
    torch.cuda.synchronize()
    ok = all(r == 0 for r in rc) and torch.equal(gath, send) and torch.equal(recv, rows)
    lib.ncclCommDestroy(comm)
    print(json.dumps({"nccl_version": ver.value, "return_codes": rc, "data_ok": bool(ok)}))
    raise SystemExit(0 if ok else 1)


if __name__ == "__main__":
    main()
