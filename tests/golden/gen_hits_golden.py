"""Record the REFERENCE keyphrase_hits (evaluation.py:110-134) on the seeded
cases of tests/hits_cases.py -> tests/golden/hits_golden.json (run in the
build container; builds the reference in a scratch copy like gen_golden.py)."""

import json
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, str(HERE))

import hits_cases as hc  # noqa: E402
from gen_golden import ensure_ref  # noqa: E402


def main():
    sys.path.insert(0, str(ensure_ref(None)))
    from phraseboost.evaluation import keyphrase_hits

    out = {}
    for seed in hc.SEEDS:
        refs, hyps, phrases, ci = hc.case(seed)
        hits = keyphrase_hits(refs, hyps, phrases, case_insensitive=ci)
        out[str(seed)] = [[k, h.ref, h.hyp, h.tp, h.fp, h.fn] for k, h in hits.items()]
    (HERE / "hits_golden.json").write_text(json.dumps(out, indent=0) + "\n")
    print("wrote", len(out), "cases")


if __name__ == "__main__":
    main()
