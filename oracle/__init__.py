"""CPU oracle for the KiloNeuS render hot path -- TEST INFRASTRUCTURE ONLY.

This package is a NumPy restatement of the reference algorithm (the
``kilofield`` package mounted at /root/reference/pkg/src/kilofield) for the
one hot path this repository accelerates.  Every function cites the reference
file:line it follows.  It is the *checker*: only ``tests/``,
``__graft_entry__.smoke()`` and the ``cpu_baseline`` / ``--impl reference``
legs of ``bench.py`` may import it.  The product package
(``paper_2206_10885_b200``) never imports, links or executes anything here and
has no CPU fallback.

Pinning status: PINNED.  The reference is pure Python/NumPy, so it was
imported in the build container and run on seeded inputs by
``tests/golden/make_golden.py``; the resulting vectors are committed under
``tests/golden/`` and ``tests/test_oracle_golden.py`` checks this restatement
against them (cell ids, RNG and step counts exactly; floating-point outputs to
<= 2e-6, and bit-for-bit on the machine that generated them).  The reference
holds no stored golden vectors of its own; its known-answer tests for the path
(cell corners, ray/AABB cases, furnace exactness -- SURVEY.md section 8c) are
re-run against this oracle in ``tests/test_oracle_known_answers.py``.

One piece is C: ``oracle/np_softplus.c`` restates, operation for operation, how NumPy 2.3 evaluates the float32
softplus of nn.py:26-33 on an AVX-512 host (np.exp's source loop + Intel SVML's log1p, a third-party routine pinned to
the installed numpy binary); ``tests/test_oracle_golden.py::test_softplus_restatement_bit_exact`` checks it against
NumPy itself and against the reference-generated golden vector.  It documents the arithmetic the device softplus
reproduces; like everything here it is only ever run by the tests.

Arithmetic note: like the reference, the oracle's matrix products go through
NumPy -> OpenBLAS ``sgemm`` and its transcendentals through NumPy's SIMD loops,
so last-ulp results depend on the host CPU and on how many points share a cell
(OpenBLAS switches kernels by problem size).  DESIGN.md section "Numerics"
measures that noise floor.
"""

from .field import (  # noqa: F401
    FieldSpec,
    FieldParams,
    OracleField,
    make_random_field,
    positional_features,
    softplus32,
    logistic32,
    cell_triples,
    cell_ids,
    group_by_cell,
    grouped_forward,
    query_sdf,
    query_sdf_values,
    query_color,
    grouped_query,
    fd_probe_points,
    fd_gradient,
    fd_normals,
)
from .trace import (  # noqa: F401
    Camera,
    camera_look_at,
    camera_rays,
    MarchSettings,
    FieldTraceable,
    slab_intersect,
    march,
    trace_shade,
    render,
    pass_image,
)
from .volume import volume_forward  # noqa: F401
from .paths import (  # noqa: F401
    hash_uniform,
    SphereShape,
    QuadShape,
    BoxShape,
    NeuralShape,
    Diffuse,
    Emitter,
    UniformSky,
    PathScene,
    tangent_frame,
    cosine_sample,
    nearest_hit,
    trace_paths,
    render_paths,
)
