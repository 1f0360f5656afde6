"""Per-task execution times of a saved PASE_TRACE timeline (gpurun_out/trace_<workload>.npy):
end - max(start, last warp's gate opening), us, float64 in task-id order -> argv[2]
(for the PASE_DUR_FILE list-schedule A/B)."""
import sys

import numpy as np

tr = np.load(f"gpurun_out/trace_{sys.argv[1]}.npy")
seen = tr[:, 7:23:2]
gs = np.where(seen > 0, seen, 0).max(1)
ex = (tr[:, 6] - np.maximum(tr[:, 3], gs)) / 1e3
ex = np.where(tr[:, 0] >= 0, np.maximum(ex, 0.5), 0.0)
ex.astype(np.float64).tofile(sys.argv[2])
print(sys.argv[1], len(ex), "tasks, mean %.2f us" % ex.mean())
