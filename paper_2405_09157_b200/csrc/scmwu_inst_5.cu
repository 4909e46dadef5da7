// scmwu_inst_5.cu — explicit instantiations of the persistent kernel (part 5 of 8).
#include "scmwu_kernel.cuh"

SCMWU_INST(SC_SVM, 4, 3)
SCMWU_INST(SC_SVM, 8, 6)
SCMWU_INST(SC_SVM, 8, 16)
SCMWU_INST(SC_SVM, 32, 16)

namespace scmwu {
KernelFn scmwu_lookup_5(int kind, int lpr, int cpl) {
    SCMWU_MATCH(SC_SVM, 4, 3)
    SCMWU_MATCH(SC_SVM, 8, 6)
    SCMWU_MATCH(SC_SVM, 8, 16)
    SCMWU_MATCH(SC_SVM, 32, 16)
    return nullptr;
}
}  // namespace scmwu
