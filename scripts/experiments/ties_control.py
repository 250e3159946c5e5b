# control: the drop-in beams with the top-k tie group disabled (plain k cut)
import sys
import pytest
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from paper_2508_07014_b200 import decoding as d
orig = d._TopK.__call__
def plain(self, rows_dev, ld, states, am, boost, exclude, k, alt_token=None, alt_am=None, valid=None, skip_neg_inf=False):
    k = min(int(k), len(am) * self.V)
    return self._run(rows_dev, ld, states, am, boost, exclude, k, alt_token, alt_am, valid, skip_neg_inf)
d._TopK.__call__ = plain
sys.exit(pytest.main(["tests/test_ties.py", "-q", "-m", "gpu", "-p", "no:cacheprovider"]))
