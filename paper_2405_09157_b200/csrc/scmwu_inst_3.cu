// scmwu_inst_3.cu — explicit instantiations of the persistent kernel (part 3 of 8).
#include "scmwu_kernel.cuh"

SCMWU_INST(SC_SES, 2, 4, 2, false)
SCMWU_INST(SC_SVM, 4, 4, 4, false)
SCMWU_INST(SC_SES, 8, 6, 4, true)
SCMWU_INST(SC_SES, 8, 13, 4, false)
SCMWU_INST(SC_SVM, 16, 12, 2, false)
SCMWU_INST(SC_SES, 32, 16, 2, true)

namespace scmwu {
KernelFn scmwu_lookup_3(int kind, int lpr, int cpl, int nb, bool full) {
    SCMWU_MATCH(SC_SES, 2, 4, 2, false)
    SCMWU_MATCH(SC_SVM, 4, 4, 4, false)
    SCMWU_MATCH(SC_SES, 8, 6, 4, true)
    SCMWU_MATCH(SC_SES, 8, 13, 4, false)
    SCMWU_MATCH(SC_SVM, 16, 12, 2, false)
    SCMWU_MATCH(SC_SES, 32, 16, 2, true)
    return nullptr;
}
}  // namespace scmwu
