// scmwu_inst_0.cu — explicit instantiations of the persistent kernel (part 0 of 8).
#include "scmwu_kernel.cuh"

SCMWU_INST(SC_SES, 2, 2, 2, false)
SCMWU_INST(SC_SVM, 4, 3, 4, false)
SCMWU_INST(SC_SES, 4, 8, 4, true)
SCMWU_INST(SC_SES, 8, 10, 4, false)
SCMWU_INST(SC_SVM, 8, 16, 2, false)
SCMWU_INST(SC_SES, 32, 12, 2, true)

namespace scmwu {
KernelFn scmwu_lookup_0(int kind, int lpr, int cpl, int nb, bool full) {
    SCMWU_MATCH(SC_SES, 2, 2, 2, false)
    SCMWU_MATCH(SC_SVM, 4, 3, 4, false)
    SCMWU_MATCH(SC_SES, 4, 8, 4, true)
    SCMWU_MATCH(SC_SES, 8, 10, 4, false)
    SCMWU_MATCH(SC_SVM, 8, 16, 2, false)
    SCMWU_MATCH(SC_SES, 32, 12, 2, true)
    return nullptr;
}
}  // namespace scmwu
