"""Generate tests/golden/*.json from the reference itself (oracle/_ref).

Run here (where /root/reference exists and `make oracle` has built
oracle/_ref/libeps_ref.so).  The GPU box never reads /root/reference: tests
there use the committed fixtures this script writes.

    python tests/golden/make_golden.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from paper_2102_03161_b200 import configs  # noqa: E402
from paper_2102_03161_b200.capi import EpsApi  # noqa: E402

REF_CONFIGS = "/root/reference/proj/configs"


def main():
    ref = EpsApi(os.path.join(ROOT, "oracle/_ref/libeps_ref.so"), "epsref_")
    out = {"scenarios": []}
    cases = []
    for name in ("vit_reference", "bert_reference", "ideal_multiplicative"):
        # re-serialised through the reference's own scenario_to_json
        cases.append((name, ref.scenario(os.path.join(REF_CONFIGS, name + ".json")).to_json()))
    for cid in configs.BASELINE_CONFIGS:
        for g in ((1,) if cid == "tiny-vit" else (1, 2, 4, 8)):
            cases.append((f"{cid}-g{g}", configs.scenario(cid, g)))
            cases.append((f"{cid}-g{g}-nofreeze", configs.no_freeze(configs.scenario(cid, g))))
    for name, scen in cases:
        s = ref.scenario(scen)
        rows, summ = s.simulate()
        out["scenarios"].append({
            "name": name,
            "scenario": scen,
            "rows": rows,
            "summary": summ,
            "report_csv": s.report(0),
            "transitions_jsonl": s.report(3),
            "breakdown": s.speedup_breakdown() if name == "vit_reference" else None,
        })
    path = os.path.join(ROOT, "tests/golden/decisions.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print("wrote", path, len(out["scenarios"]), "scenarios")


if __name__ == "__main__":
    main()
