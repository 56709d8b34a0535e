// Instantiations of every kernel for one dtype (DT_I32); compiled in parallel
// with the other dtypes (see build.py).
#include "kernels.cuh"

namespace stragglar {

void* select_kernel_i32(int which, int world, int mover) {
  switch (world) {
    case 2: return kernel_ptr<DT_I32, 2>(which, mover);
    case 4: return kernel_ptr<DT_I32, 4>(which, mover);
    case 6: return kernel_ptr<DT_I32, 6>(which, mover);
    case 8: return kernel_ptr<DT_I32, 8>(which, mover);
    default: return nullptr;
  }
}

}  // namespace stragglar
