"""B200-native low-synchronization block Arnoldi (BCGS-PIP) with restarted BFOM/BGMRES.

Lund, "Adaptively restarted block Krylov subspace methods with low-synchronization
skeletons", arXiv 2208.09899.  The compute path is hand-written sm_100a CUDA behind the C ABI
in include/lsba.h (liblsba.so, built in-tree by ``__graft_entry__.build()``); this package is a
thin ctypes binding with the same names.  There is no CPU fallback: importing the binding
raises if liblsba.so is missing.
"""
from ._lib import (  # noqa: F401
    LsbaError,
    SolveInfo,
    StepInfo,
    Context,
    lib,
    library_path,
    LSBA_IP_CLASSICAL,
    LSBA_IP_GLOBAL,
    LSBA_SKEL_BCGS_PIP,
    LSBA_SKEL_BMGS_CWY,
    LSBA_SKEL_BMGS_ICWY,
    LSBA_SKEL_BMGS,
    LSBA_SKEL_BCGS_PIO,
    LSBA_SKEL_BCGS_IROLS,
    LSBA_CONVERGED,
    LSBA_MAX_RESTARTS,
    LSBA_DEAD,
    KERNEL_IDS,
    lsba_get_unique_id,
    lsba_create,
    lsba_destroy,
    lsba_arnoldi_begin,
    lsba_block_arnoldi_step,
    lsba_copy_hessenberg,
    lsba_projected_solve,
    lsba_copy_beta,
    lsba_copy_basis_block,
    lsba_bgmres_solve,
    lsba_bfom_solve,
    lsba_solve_host,
    lsba_spmm,
    lsba_block_inner_product,
    lsba_set_force_flag,
    lsba_set_kernel_variant,
    lsba_set_skeleton,
    lsba_profile_enable,
    lsba_profile_read,
    lsba_profile_timeline,
    lsba_launch_count,
    lsba_workspace_bytes,
    lsba_ghost_plan,
    lsba_csr_validate,
    lsba_status_str,
    lsba_last_error,
)
