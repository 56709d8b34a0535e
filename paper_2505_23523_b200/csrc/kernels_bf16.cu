// Instantiations of every kernel for one dtype (DT_BF16); compiled in parallel
// with the other dtypes (see build.py).
#include "kernels.cuh"

namespace stragglar {

void* select_kernel_bf16(int which, int world, int mover) {
  switch (world) {
    case 2: return kernel_ptr<DT_BF16, 2>(which, mover);
    case 4: return kernel_ptr<DT_BF16, 4>(which, mover);
    case 6: return kernel_ptr<DT_BF16, 6>(which, mover);
    case 8: return kernel_ptr<DT_BF16, 8>(which, mover);
    default: return nullptr;
  }
}

}  // namespace stragglar
