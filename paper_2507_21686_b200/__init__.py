"""paper_2507_21686_b200 -- B200 (sm_100a) evaluator of analytic SPH boundary
integrals over triangles (arXiv 2507.21686), drop-in for the reference's
`sphbi::integrate_triangle` hot path. See DESIGN.md."""
from . import sphbi  # noqa: F401
from .sphbi import (  # noqa: F401
    Context, DomainError, IntegralResult, InvalidArgument, KernelTermTable, LogicError, Point2, PolyKernel,
    SingularInput, Triangle, UnsupportedForm, default_context, evaluate, integrate_pairs, integrate_triangle,
    integrate_triangle_bases, kernel_by_name, table1_terms, wendland4)
