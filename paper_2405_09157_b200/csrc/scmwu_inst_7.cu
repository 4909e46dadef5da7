// scmwu_inst_7.cu — explicit instantiations of the persistent kernel (part 7 of 8).
#include "scmwu_kernel.cuh"

SCMWU_INST(SC_SVM, 4, 4, 4)
SCMWU_INST(SC_SVM, 8, 8, 4)
SCMWU_INST(SC_SVM, 16, 12, 2)

namespace scmwu {
KernelFn scmwu_lookup_7(int kind, int lpr, int cpl, int nb) {
    SCMWU_MATCH(SC_SVM, 4, 4, 4)
    SCMWU_MATCH(SC_SVM, 8, 8, 4)
    SCMWU_MATCH(SC_SVM, 16, 12, 2)
    return nullptr;
}
}  // namespace scmwu
