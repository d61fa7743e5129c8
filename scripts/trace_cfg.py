"""Per-phase trace of the CTA that runs item 0 of each device step (development aid).
Times in ns relative to the end of the previous step (max over CTAs of its last item)."""
import sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np, torch
import workloads as W
from harness import run_gpu
from paper_2302_03851_b200 import edbatch as E
name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
wl = W.config(name)
plan, w, ws, out = run_gpu(wl)
nb = plan.info["num_steps"]
tr = torch.zeros(nb * 64 + 148 * 4, dtype=torch.int64, device="cuda")
for _ in range(3):
    tr.zero_()
    E.ed_execute(plan, w, ws, out, trace=tr)
torch.cuda.synchronize()
full = tr.cpu().numpy().astype(np.int64)
t = full[:nb * 64].reshape(nb, 64)
pc = full[nb * 64:].reshape(148, 4)
i = ws.plan_info
ts = ws._view(i["off_ts"], nb + 1, torch.int64).cpu().numpy().astype(np.int64)
end = np.maximum.accumulate(ts)
sched = plan.schedule()
print("phases rel. to previous step end (ns): reached, rows-ready, A-issued, MMA-1st-full, MMA-issued, EPI-got-acc, EPI-done | step end")
for s in range(nb):
    base = end[s]
    rel = lambda k: int(t[s, k] - base) if t[s, k] else None
    print(s, len(sched[min(s, len(sched) - 1)][1]), [rel(k) for k in (0, 1, 2, 3, 4, 6, 5)], "|", int(ts[s + 1] - base),
          " epi loop/fence/publish:", [rel(k) for k in (7, 8, 9)])

# per-CTA SIMT (last step) phases: entered, passed the CTA barrier, items done (rel. to previous step end)
base = end[nb - 1]
rows = [(c, int(pc[c, 0] - base), int(pc[c, 1] - base), int(pc[c, 2] - base)) for c in range(148) if pc[c, 1]]
rows.sort(key=lambda r: -r[3])
print("last step per CTA (cta, enter, synced, done) slowest first:", rows[:12])
print("median enter/synced/done:", [int(np.median([r[k] for r in rows])) for k in (1, 2, 3)])
it = [(c, int(pc[c, 1] - base), int(pc[c, 0] - base), int(pc[c, 3] - base) if pc[c, 3] else None, int(pc[c, 2] - base)) for c in range(148) if pc[c, 1]]
it.sort(key=lambda r: -r[4])
print("per CTA (cta, synced, item1 done, item2 done, all done) slowest first:", it[:16])
print("fastest:", it[-6:])

# first step (device step 0): per-CTA item completion times (slots 0..2) and item count (slot 3)
print("step 0 per-CTA item ends (us after kernel start), by number of items:")
t0k = int(ts[0])
by = {}
for c in range(148):
    n = int(pc[c, 3])
    if n <= 0 or n > 3:
        continue
    ends = [round((int(pc[c, k]) - t0k) / 1e3, 1) for k in range(min(n, 3))]
    by.setdefault(n, []).append(ends)
for n, rows in sorted(by.items()):
    arr = np.array(rows)
    print(f"  {n} items: {len(rows)} CTAs; item-end medians {np.median(arr, axis=0).tolist()}; max last {arr[:, -1].max()}")
