// scmwu_inst_6.cu — explicit instantiations of the persistent kernel (part 6 of 8).
#include "scmwu_kernel.cuh"

SCMWU_INST(SC_SES, 4, 3, 4, false)
SCMWU_INST(SC_SVM, 4, 6, 4, false)
SCMWU_INST(SC_SES, 8, 8, 4, true)
SCMWU_INST(SC_SES, 8, 16, 2, false)
SCMWU_INST(SC_SVM, 16, 16, 2, false)

namespace scmwu {
KernelFn scmwu_lookup_6(int kind, int lpr, int cpl, int nb, bool full) {
    SCMWU_MATCH(SC_SES, 4, 3, 4, false)
    SCMWU_MATCH(SC_SVM, 4, 6, 4, false)
    SCMWU_MATCH(SC_SES, 8, 8, 4, true)
    SCMWU_MATCH(SC_SES, 8, 16, 2, false)
    SCMWU_MATCH(SC_SVM, 16, 16, 2, false)
    return nullptr;
}
}  // namespace scmwu
