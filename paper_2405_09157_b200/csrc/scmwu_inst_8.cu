// scmwu_inst_8.cu — explicit instantiations of the persistent kernel (part 8): smaller
// warp tiles (fewer row-groups per batch, so more ring stages fit in shared memory).
#include "scmwu_kernel.cuh"

SCMWU_INST(SC_SES, 8, 13, 2, true)
SCMWU_INST(SC_SVM, 8, 13, 2, false)
SCMWU_INST(SC_SES, 32, 16, 1, true)
SCMWU_INST(SC_SVM, 32, 16, 1, false)
SCMWU_INST(SC_SVM, 16, 32, 2, false)

namespace scmwu {
KernelFn scmwu_lookup_8(int kind, int lpr, int cpl, int nb, bool full) {
    SCMWU_MATCH(SC_SES, 8, 13, 2, true)
    SCMWU_MATCH(SC_SVM, 8, 13, 2, false)
    SCMWU_MATCH(SC_SES, 32, 16, 1, true)
    SCMWU_MATCH(SC_SVM, 32, 16, 1, false)
    SCMWU_MATCH(SC_SVM, 16, 32, 2, false)
    return nullptr;
}
}  // namespace scmwu
