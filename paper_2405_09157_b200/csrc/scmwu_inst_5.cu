// scmwu_inst_5.cu — explicit instantiations of the persistent kernel (part 5 of 8).
#include "scmwu_kernel.cuh"

SCMWU_INST(SC_SVM, 4, 3, 4)
SCMWU_INST(SC_SVM, 8, 6, 4)
SCMWU_INST(SC_SVM, 8, 16, 2)
SCMWU_INST(SC_SVM, 32, 16, 2)

namespace scmwu {
KernelFn scmwu_lookup_5(int kind, int lpr, int cpl, int nb) {
    SCMWU_MATCH(SC_SVM, 4, 3, 4)
    SCMWU_MATCH(SC_SVM, 8, 6, 4)
    SCMWU_MATCH(SC_SVM, 8, 16, 2)
    SCMWU_MATCH(SC_SVM, 32, 16, 2)
    return nullptr;
}
}  // namespace scmwu
