"""Record the REFERENCE's own blend-stage output as golden fixtures (run in the build container,
where /root/reference exists; the fixtures are committed and travel without it).

For each case below: write the dataset shards as JSONL ({"doc_id", "dataset", "text"}), a pipeline
config with stages ["blend"], run the reference curator pipeline (oracle/_ref/ref_pipeline, compiled
unmodified from /root/reference/proj/src by oracle/Makefile) and copy its
<work_dir>/blend/blend_manifest.jsonl to tests/golden/blend/<case>.jsonl. cases.json records the
inputs so tests/test_feed.py can regenerate each manifest through mt_blend_manifest and compare
bytes.

    python tests/golden/make_blend_golden.py
"""
from __future__ import annotations

import json
import subprocess
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
OUT = Path(__file__).resolve().parent / "blend"

# name -> (datasets [(name, weight, doc ids)], batch_size, steps, shuffle, seed)
CASES = {
    "three_in_order": ([("web", 0.5, list(range(0, 40))), ("books", 0.3, list(range(100, 125))),
                        ("code", 0.2, list(range(500, 510)))], 16, 12, False, 0),
    "three_shuffled": ([("web", 0.5, list(range(0, 40))), ("books", 0.3, list(range(100, 125))),
                        ("code", 0.2, list(range(500, 510)))], 16, 12, True, 7),
    # percentage weights (normalised by the stage), config order != name order, sparse doc ids
    "percent_mix": ([("zeta", 14.3, [1000 + 3 * i for i in range(30)]), ("alpha", 19.3, [5000 + i for i in range(7)]),
                     ("mid", 5.7, [9000 + 11 * i for i in range(50)]), ("beta", 2.9, [20000 + i for i in range(3)]),
                     ("omega", 4.8, [30000 + 2 * i for i in range(12)])], 32, 20, True, 11),
    # non-ASCII and escaped characters in a dataset name go through the JSON writer
    "escaped_name": ([("wiki-ü \"q\"", 0.25, list(range(0, 9))), ("plain", 0.75, list(range(50, 80)))],
                     8, 10, True, 3),
}


def main() -> None:
    subprocess.run(["make", "-s", "-C", str(ROOT / "oracle"), "_ref/ref_pipeline"], check=True)
    exe = ROOT / "oracle" / "_ref" / "ref_pipeline"
    OUT.mkdir(parents=True, exist_ok=True)
    meta = {}
    with tempfile.TemporaryDirectory() as tmp:
        tmp = Path(tmp)
        for case, (datasets, batch, steps, shuffle, seed) in CASES.items():
            cfg_ds = []
            for k, (name, weight, ids) in enumerate(datasets):
                path = tmp / f"{case}_{k}.jsonl"
                with open(path, "w", encoding="utf-8") as f:
                    for i in ids:
                        f.write(json.dumps({"doc_id": i, "dataset": name, "text": f"document {i}"},
                                           ensure_ascii=False) + "\n")
                cfg_ds.append({"name": name, "weight": weight, "path": str(path)})
            cfg = {"seed": seed, "work_dir": str(tmp / f"work_{case}"), "stages": ["blend"], "datasets": cfg_ds,
                   "blend": {"batch_size": batch, "steps": steps, "shuffle": shuffle}}
            cfg_path = tmp / f"{case}.json"
            cfg_path.write_text(json.dumps(cfg, ensure_ascii=False), encoding="utf-8")
            r = subprocess.run([str(exe), str(cfg_path)], capture_output=True, text=True)
            if r.returncode:
                sys.exit(f"{case}: reference pipeline failed: {r.stderr}")
            manifest = (tmp / f"work_{case}" / "blend" / "blend_manifest.jsonl").read_bytes()
            (OUT / f"{case}.jsonl").write_bytes(manifest)
            meta[case] = {"datasets": [{"name": n, "weight": w, "doc_ids": ids} for n, w, ids in datasets],
                          "batch_size": batch, "steps": steps, "shuffle": shuffle, "seed": seed}
            print(f"{case}: {manifest.count(b'\n')} lines")
    (OUT / "cases.json").write_text(json.dumps(meta, indent=1, ensure_ascii=False) + "\n", encoding="utf-8")


if __name__ == "__main__":
    main()
