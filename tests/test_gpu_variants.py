"""Every tuning switch of DESIGN §6.1 keeps the results bit-exact: the parity checks of
tests/test_gpu_parity.py re-run in a subprocess per switch setting (the switches are read once
per process).  Forcing the single-suffix 2-D forms, the wave tail and the widening onto small
graphs exercises code paths the default plans reserve for the big zoo vertices."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

VARIANTS = {
    "2s_everywhere": {"PASE_MIN_2S": "0"},
    "no_2d": {"PASE_NO_2D": "1"},
    "no_latency_mode": {"PASE_LATENCY_CAND": "0"},
    "narrow_groups": {"PASE_C_PER_LANE": "8"},
    "no_tail_no_widen": {"PASE_WAVE_TAIL": "0", "PASE_WIDEN": "0"},
    "cost_tasks": {"PASE_COST_TASKS": "1"},
    "streaming_everywhere": {"PASE_STREAM_MB": "0"},     # every spanning child -> stream tile (L2 prefetch)
    "streaming_smem_ring": {"PASE_STREAM_MB": "0", "PASE_STREAM_TMA": "1"},  # ... TMA smem ring
    "streaming_no_tma": {"PASE_STREAM_MB": "0", "PASE_STREAM_TMA": "0"},   # ... or plain full-warp 1-D tile
    "ready_queue": {"PASE_QUEUE": "1"},                   # ready-queue claiming instead of the static order
    "cta_gate": {"PASE_EARLY_GATE": "0"},                 # one thread per CTA waits before the tile
    "elected_gate_no_warm": {"PASE_GATE_ELECT": "1", "PASE_WARM": "0"},   # one poller per CTA, no warm pass
    "task_length_cap": {"PASE_MAX_LANE_CAND": "64"},      # every big vertex widened (more, shorter tasks)
    "fitted_durations": {"PASE_DUR": "1:3.4:2500,2:4:9000,3:3.3:3500,4:5:8500"},   # another claim order
    "cta_tile": {"PASE_CTA": "1"},                        # CTA-tiled min-plus for the big vertices
    "gate_fence": {"PASE_GATE_LDACQ": "0"},               # gates acquire by fence.acq_rel (round-1 form)
    "gate_ldacq_1d": {"PASE_GATE_LDACQ": "1"},            # ld.acquire at 1-D tile gates only
    "release_atom": {"PASE_REL_RED": "0"},                # releases by atom.acq_rel (round-1 form)
    "latency_two_c_per_lane": {"PASE_LAT_ONE_TASKS": "0"},   # no one-C-per-lane latency groups
}


@pytest.mark.parametrize("variant", sorted(VARIANTS))
def test_switch_keeps_parity(variant):
    env = dict(os.environ)
    env.update(VARIANTS[variant])
    env["PYTHONPATH"] = ROOT + os.pathsep + env.get("PYTHONPATH", "")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "parity_variant_main.py"),
                        "mlp,alexnet,inception_v3,transformer", "12"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "variant parity ok" in r.stdout, (r.stdout + r.stderr)[-3000:]
