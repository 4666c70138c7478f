#!/usr/bin/env python3
"""Write the BASELINE configs as scene files in the reference's schema
(scene.py; SURVEY.md §8d-4 "Freeze this scene as a JSON file"):

  scenes/config4.json          the headline scene, random-init paper models (scenes/models/, generated)
  scenes/config5.json          config 4 + the dynamic spin as keyframe tracks
  scenes/config4_trained.json  config-4 placements with the distilled fixtures (tests/golden/trained_*.nedm)
"""

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2308_04669_b200 import configs as CF, scene as S  # noqa: E402

OUT = ROOT / "scenes"


def main():
    OUT.mkdir(exist_ok=True)
    spec = CF.config4()
    rand = lambda o: f"models/{S.model_file_name(o.kind, o.seed)}"      # noqa: E731
    trained = lambda o: f"../tests/golden/trained_{o.kind}.nedm"         # noqa: E731
    docs = {"config4.json": S.scene_document(spec, rand),
            "config5.json": S.scene_document(spec, rand, animation=CF.config5_keyframes()),
            "config4_trained.json": S.scene_document(spec, trained)}
    for name, doc in docs.items():
        (OUT / name).write_text(json.dumps(doc, indent=2) + "\n")
        print("wrote", OUT / name)


if __name__ == "__main__":
    main()
