"""What the bench's L2 flush between closed loops costs on C2: device time
per ADMM iteration over seeds 1..20 (one loop each, like bench.py), with and
without a 256 MiB write before every loop; alternated 3 times."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch
import paper_2103_14990_b200 as pb
system = pb.build_chain_network(100)
spec = pb.make_benchmark_spec(system, 10)
mask = pb.build_locality_mask(system, 3, 10)
sess = pb.DlmpcSession(system, spec, mask, "b200")
dev = sess.device
xs = [torch.tensor(pb.sample_initial_state(system.partition, np.random.default_rng(s)), dtype=torch.float64,
                   device="cuda:0") for s in range(1, 21)]
states = torch.zeros(21 * 200, dtype=torch.float64, device="cuda:0")
inputs = torch.zeros(20 * 100, dtype=torch.float64, device="cuda:0")
iters = torch.zeros((20, 20), dtype=torch.int32, device="cuda:0")
status = torch.zeros((20, 8), dtype=torch.int32, device="cuda:0")
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda:0")
ext = torch.cuda.ExternalStream(dev.stream, device="cuda:0")
for rep in range(3):
    for fl in (True, False):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
        for k in range(20):
            if fl:
                flush.zero_()
            torch.cuda.synchronize()
            ev[k][0].record(ext)
            dev.simulate_device(xs[k].data_ptr(), 20, spec.max_iters, spec.eps_pri, spec.eps_dual, states.data_ptr(),
                                inputs.data_ptr(), iters[k].data_ptr(), status[k].data_ptr())
            ev[k][1].record(ext)
        torch.cuda.synchronize()
        ms = sum(a.elapsed_time(b) for a, b in ev)
        it = int(iters.sum())
        print(f"flush={fl}: {1e3 * ms / it:.3f} us/iter  {100 * it / (ms * 1e-3) / 1e6:.3f} M subsystem-iters/s", flush=True)
