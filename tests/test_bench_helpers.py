"""bench.py's host-side helpers (CPU): the library reference point it
copies into its line from the committed same-box capture, and the bounded
CPU sample of the reference arm."""
from __future__ import annotations

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402


def test_library_reference_cites_its_capture():
    ref = bench.library_reference("cfg2")
    assert ref is not None and ref["source"] == "profiles/r02_library_baseline_cfg2.json"
    raw = json.loads((ROOT / ref["source"]).read_text().strip().splitlines()[-1])
    # the numbers are the capture's own, not re-derived
    assert ref["ours_us"] == raw["ours"]["us"]
    assert ref["cascade_us"] == raw["cascade"]["us"] and ref["trtllm_gen_decode_us"] == raw["trtllm_gen_decode"]["us"]
    # both library arms agree with this path's output within the bf16 bar
    assert ref["cascade_max_abs_vs_ours"] < 2e-3 and ref["trtllm_gen_decode_max_abs_vs_ours"] < 2e-3


def test_library_reference_absent_for_other_configs():
    assert bench.library_reference("cfg3") is None


def test_reference_sample_is_bounded():
    """The CPU arm times kv heads [0, ref_heads) of the whole workload
    (cfg4: trees 0..7 only), so its run ends within minutes."""
    for name in ("cfg2", "cfg4", "cfg5"):
        cfg = dict(bench.CONFIGS[name], name=name)
        spec, hk, desc = bench._ref_sample_spec(cfg)
        assert hk <= cfg["h_kv"] and "kv heads" in desc
        assert bench._ref_bytes(spec, hk, cfg["d"]) > 0
