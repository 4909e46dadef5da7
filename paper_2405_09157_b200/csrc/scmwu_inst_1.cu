// scmwu_inst_1.cu — explicit instantiations of the persistent kernel (part 1 of 8).
#include "scmwu_kernel.cuh"

SCMWU_INST(SC_SES, 2, 2, 2, true)
SCMWU_INST(SC_SES, 4, 4, 4, false)
SCMWU_INST(SC_SVM, 4, 8, 4, false)
SCMWU_INST(SC_SES, 8, 10, 4, true)
SCMWU_INST(SC_SES, 16, 12, 2, false)
SCMWU_INST(SC_SVM, 32, 12, 2, false)

namespace scmwu {
KernelFn scmwu_lookup_1(int kind, int lpr, int cpl, int nb, bool full) {
    SCMWU_MATCH(SC_SES, 2, 2, 2, true)
    SCMWU_MATCH(SC_SES, 4, 4, 4, false)
    SCMWU_MATCH(SC_SVM, 4, 8, 4, false)
    SCMWU_MATCH(SC_SES, 8, 10, 4, true)
    SCMWU_MATCH(SC_SES, 16, 12, 2, false)
    SCMWU_MATCH(SC_SVM, 32, 12, 2, false)
    return nullptr;
}
}  // namespace scmwu
