"""Host-side profile of the e2e path (distributed_epoch + adam_step) at a config (default c3)."""
import cProfile
import pstats
import sys
import time
CFG_KEY = sys.argv[1] if len(sys.argv) > 1 else "c3"
sys.path.insert(0, ".")
import bench  # noqa: E402
import torch  # noqa: E402
import paper_2109_07893_b200 as pk  # noqa: E402

bench.select_config(CFG_KEY)
cfg, g, data, train, params = bench.make_workload(1)
nblk = bench.nblk_for(1)
hp = {k: v.copy() for k, v in params.items()}
st = pk.init_adam(hp)
for _ in range(2):
    loss, grads, _, _ = pk.distributed_epoch(cfg, data, train, hp, 1, nblk)
    pk.adam_step(hp, grads, st, 0.01)
torch.cuda.synchronize()
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
for _ in range(3):
    loss, grads, _, _ = pk.distributed_epoch(cfg, data, train, hp, 1, nblk, comm=pk.CommLedger(),
                                             transfer=pk.TransferLedger())
    pk.adam_step(hp, grads, st, 0.01)
torch.cuda.synchronize()
pr.disable()
print("ms per e2e step", (time.perf_counter() - t0) / 3 * 1e3)
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
