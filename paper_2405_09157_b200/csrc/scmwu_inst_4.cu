// scmwu_inst_4.cu — explicit instantiations of the persistent kernel (part 4 of 8).
#include "scmwu_kernel.cuh"

SCMWU_INST(SC_SES, 2, 4, 2, true)
SCMWU_INST(SC_SES, 4, 6, 4, false)
SCMWU_INST(SC_SVM, 8, 6, 4, false)
SCMWU_INST(SC_SES, 8, 13, 4, true)
SCMWU_INST(SC_SES, 16, 16, 2, false)
SCMWU_INST(SC_SVM, 32, 16, 2, false)

namespace scmwu {
KernelFn scmwu_lookup_4(int kind, int lpr, int cpl, int nb, bool full) {
    SCMWU_MATCH(SC_SES, 2, 4, 2, true)
    SCMWU_MATCH(SC_SES, 4, 6, 4, false)
    SCMWU_MATCH(SC_SVM, 8, 6, 4, false)
    SCMWU_MATCH(SC_SES, 8, 13, 4, true)
    SCMWU_MATCH(SC_SES, 16, 16, 2, false)
    SCMWU_MATCH(SC_SVM, 32, 16, 2, false)
    return nullptr;
}
}  // namespace scmwu
