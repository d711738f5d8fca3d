import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")


def golden(name):
    return np.load(os.path.join(GOLDEN, name))


@pytest.fixture(scope="session")
def golden_dir():
    return GOLDEN


def oracle_from_product(field):
    """Wrap a product/reference-style KiloField's stacks as an OracleField (no copy)."""
    import oracle
    from oracle.field import field_from_stacks

    c = field.config
    spec = oracle.FieldSpec(resolution=c.resolution, lo=tuple(c.bbox_min), hi=tuple(c.bbox_max), pos_octaves=c.sdf_freqs,
                            dir_octaves=c.dir_freqs, n_features=c.feature_dim, fd_step=c.fd_step)
    return field_from_stacks(spec, field.sdf.weights, field.sdf.biases, field.color.weights, field.color.biases)


@pytest.fixture(scope="session")
def distilled_field():
    from paper_2206_10885_b200.modelio import load_model

    return load_model(os.path.join(GOLDEN, "sphere_r4_distilled.knf"))


@pytest.fixture(scope="session")
def distilled_oracle(distilled_field):
    return oracle_from_product(distilled_field)


@pytest.fixture(scope="session")
def small_oracle():
    """The reference tests' small_field: 4^3, seed 7 (pkg/tests/conftest.py:13-16)."""
    import oracle

    return oracle.make_random_field(oracle.FieldSpec(resolution=4), seed=7)


@pytest.fixture(scope="session")
def small_field():
    from paper_2206_10885_b200.grid import GridConfig, field_init

    return field_init(GridConfig(resolution=4), seed=7)


@pytest.fixture(scope="session")
def trained_field():
    """8^3 field distilled for 12 000 steps with the reference's own training code (tests/golden/make_trained.py)."""
    from paper_2206_10885_b200.modelio import load_model

    return load_model(os.path.join(GOLDEN, "sphere_stripes_r8_distilled.knf"))
