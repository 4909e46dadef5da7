// scmwu_inst_8.cu — explicit instantiations of the persistent kernel (part 8): SVM kernels
// with compile-time column guards for the BASELINE dimensions (d = 10, 100, 512).  Without
// them every column slot carries a runtime predicate, which the compiler keeps as bits of
// a register (LOP3 extraction + predicated DFMA + 2 MOVs per element; profiles/).
#include "scmwu_kernel.cuh"

SCMWU_INST(SC_SVM, 4, 3, 4, true)
SCMWU_INST(SC_SVM, 8, 13, 4, true)
SCMWU_INST(SC_SVM, 32, 16, 2, true)

namespace scmwu {
KernelFn scmwu_lookup_8(int kind, int lpr, int cpl, int nb, bool full) {
    SCMWU_MATCH(SC_SVM, 4, 3, 4, true)
    SCMWU_MATCH(SC_SVM, 8, 13, 4, true)
    SCMWU_MATCH(SC_SVM, 32, 16, 2, true)
    return nullptr;
}
}  // namespace scmwu
