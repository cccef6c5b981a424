"""Per-phase timeline of one sparse allreduce on an IPC world (diagnostics).

Build a marks-enabled library and run one rank per GPU:
  python -c "from paper_1802_08021_b200 import build; build.build(force=True, lib='/tmp/lib_marks.so', defines=['SPARCML_DEBUG_MARKS'])"
  SPARCML_LIB=/tmp/lib_marks.so python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 tools/allreduce_timeline.py
Prints, per rank, %globaltimer marks (block 0 / latest block, us after the push starts).
"""
import os, sys, struct, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1802_08021_b200 import sparcml as S, synth
dist.init_process_group("gloo")
rank, P = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
N = 1 << 24; k = 167772
streams = synth.uniform_streams(P, N, k, seed=1)
i, v = streams[rank]
it = torch.from_numpy(i.view(np.int32)).cuda(); vt = torch.from_numpy(v).cuda()
comm = S.Comm(N, k)
opts = S.make_opts(algo=S.SSAR_SPLIT_ALLGATHER, k_sum_hint=P * k)
out = S.new_out(N)
for _ in range(5):
    comm.barrier(); comm.allreduce(it, vt, N, out=out, opts=opts)
torch.cuda.synchronize(); dist.barrier()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    comm.allreduce(it, vt, N, out=out, opts=opts)
for _ in range(3):
    comm.barrier(); g.replay()
torch.cuda.synchronize(); dist.barrier()
ts = []
for _ in range(10):
    comm.barrier(); torch.cuda._sleep(100000)
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); g.replay(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b) * 1000)
dist.barrier()
# the same bracket around a graph of one trivial kernel: launch + event overhead
g0 = torch.cuda.CUDAGraph()
with torch.cuda.graph(g0):
    torch.cuda._sleep(1)
t0s = []
for _ in range(10):
    torch.cuda._sleep(100000)
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); g0.replay(); b.record(); torch.cuda.synchronize(); t0s.append(a.elapsed_time(b) * 1000)
ptr = S._lib.sparcml_comm_workspace(comm._h, rank)
buf = torch.empty(256, dtype=torch.uint8, device="cuda")
import ctypes
ctypes.CDLL(None)
hdrs = []
for o in range(0, 256, 64):
    h = S.Header(); S._check(S._lib.sparcml_read_header(ptr + 1144 + o, ctypes.byref(h), None)); hdrs.append(bytes(h))
raw = b"".join(hdrs)
t = struct.unpack("32Q", raw)
fused = os.environ.get("SPARCML_FUSED", "1") != "0"
names = {8:"start",9:"searched",11:"scattered",10:"pushed",1:"own_wait",2:"tab",0:"staged",6:"pass1",3:"merged",4:"stored",5:"sent",14:"data_wait",12:"recs",15:"copied",13:"end"} if fused else {8:"push.start",9:"push.searched",10:"push.scattered",11:"push.end",0:"own.start",1:"own.prologue",2:"own.tab",3:"own.merged",4:"own.gridsync",5:"own.written",6:"own.end",12:"cat.start",14:"cat.flags",15:"cat.copied",13:"cat.end"}
t0 = t[8]
line = f"rank {rank} graph AR median {sorted(ts)[5]:.1f} us (trivial graph {sorted(t0s)[5]:.1f}) | " + "  ".join(f"{names[i]} {(t[i]-t0)/1000:.1f}/{(t[16+i]-t0)/1000:.1f}" for i in ([8,9,11,10,1,2,0,6,3,4,5,14,12,15,13] if fused else [8,9,10,11,0,1,2,3,4,5,6,12,14,15,13]) if t[i])
allv = [None] * P
dist.all_gather_object(allv, line)
if rank == 0:
    print("\n".join(allv))
comm.close()
