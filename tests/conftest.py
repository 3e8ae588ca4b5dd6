"""Shared fixtures.  GPU tests are marked @pytest.mark.gpu and run through the
C ABI (libplanestereo_b200.so); everything else runs on the CPU."""
import glob
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) and the built CUDA library")


@pytest.fixture(scope="session")
def orc():
    import oracle

    return oracle.load_oracle()


@pytest.fixture(scope="session")
def ref():
    import oracle

    r = oracle.load_ref()
    if r is None:
        pytest.skip("oracle/_ref (compiled reference) not built")
    return r


@pytest.fixture(scope="session")
def ctx():
    import paper_1511_00758_b200 as ps

    c = ps.Context(0)
    yield c
    c.close()


def load_golden(name):
    z = np.load(os.path.join(GOLDEN, name), allow_pickle=False)
    d = {k: z[k] for k in z.files}
    d["meta"] = json.loads(str(d["meta"]))
    return d


def golden_names(prefix):
    return sorted(os.path.basename(p) for p in glob.glob(os.path.join(GOLDEN, prefix + "*.npz")))


def random_image(width, height, seed):
    """testutil::randomImage (proj/tests/testutil.hpp:10-17): raw std::mt19937(seed)
    draws & 0xff.  numpy's RandomState seeds MT19937 with init_genrand exactly like
    std::mt19937, so the images are the reference tests' own images."""
    rs = np.random.RandomState(seed)
    raw = rs.randint(0, 2**32, size=width * height, dtype=np.uint32)
    return (raw & 0xFF).astype(np.uint8).reshape(height, width)


def config_of(meta):
    import paper_1511_00758_b200 as ps

    return ps.PipelineConfig(**meta["config"])
