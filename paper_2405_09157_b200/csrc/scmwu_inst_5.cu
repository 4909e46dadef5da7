// scmwu_inst_5.cu — explicit instantiations of the persistent kernel (part 5 of 8).
#include "scmwu_kernel.cuh"

SCMWU_INST(SC_SVM, 2, 4, 2, false)
SCMWU_INST(SC_SES, 4, 6, 4, true)
SCMWU_INST(SC_SES, 8, 8, 4, false)
SCMWU_INST(SC_SVM, 8, 13, 4, false)
SCMWU_INST(SC_SES, 16, 16, 2, true)

namespace scmwu {
KernelFn scmwu_lookup_5(int kind, int lpr, int cpl, int nb, bool full) {
    SCMWU_MATCH(SC_SVM, 2, 4, 2, false)
    SCMWU_MATCH(SC_SES, 4, 6, 4, true)
    SCMWU_MATCH(SC_SES, 8, 8, 4, false)
    SCMWU_MATCH(SC_SVM, 8, 13, 4, false)
    SCMWU_MATCH(SC_SES, 16, 16, 2, true)
    return nullptr;
}
}  // namespace scmwu
