"""B200-native SCMWU feasibility engine (arXiv 2405.09157 hot path).

Modules mirror the reference package ``symcone``:
    config     RunConfig
    cones      cone shape descriptors
    meta       feasibility tests (one persistent CUDA kernel per test) and the
               host-side adaptive search
    ses        smallest enclosing sphere solver
    svm        hard-margin SVM / polytope distance solver
    instances  generators, text / .npz / memory-mapped .npyd instance files
    baselines  the reference's verification solvers (MEB, Gilbert) on the GPU
    report     run reports, verification and sweeps (the reference's bench driver)
    devgen     instances drawn directly in HBM (C4 / C5 scale)
    shard      row sharding across GPUs (one process per GPU)
The compute path is ``libscmwu.so`` (CUDA, sm_100a) behind include/scmwu.h.
"""
from . import baselines, config, cones, devgen, instances, meta, report, ses, shard, svm  # noqa: F401
from .config import RunConfig  # noqa: F401
from .ses import SesInstance, SesSolution, solve_ses  # noqa: F401
from .svm import InfeasibleInputError, SvmInstance, SvmSolution, solve_svm  # noqa: F401

__version__ = "0.1.0"
