// scmwu_inst_2.cu — explicit instantiations of the persistent kernel (part 2 of 8).
#include "scmwu_kernel.cuh"

SCMWU_INST(SC_SVM, 2, 2, 2, false)
SCMWU_INST(SC_SES, 4, 4, 4, true)
SCMWU_INST(SC_SES, 8, 6, 4, false)
SCMWU_INST(SC_SVM, 8, 10, 4, false)
SCMWU_INST(SC_SES, 16, 12, 2, true)
SCMWU_INST(SC_SES, 32, 16, 2, false)

namespace scmwu {
KernelFn scmwu_lookup_2(int kind, int lpr, int cpl, int nb, bool full) {
    SCMWU_MATCH(SC_SVM, 2, 2, 2, false)
    SCMWU_MATCH(SC_SES, 4, 4, 4, true)
    SCMWU_MATCH(SC_SES, 8, 6, 4, false)
    SCMWU_MATCH(SC_SVM, 8, 10, 4, false)
    SCMWU_MATCH(SC_SES, 16, 12, 2, true)
    SCMWU_MATCH(SC_SES, 32, 16, 2, false)
    return nullptr;
}
}  // namespace scmwu
