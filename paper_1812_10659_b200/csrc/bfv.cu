#include "bfv.hpp"

namespace lb {

void bfv_setup(Context& cx) { cx.bfv_ = std::make_unique<BfvState>(); }

}  // namespace lb
