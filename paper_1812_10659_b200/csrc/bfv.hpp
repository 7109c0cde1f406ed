// BFV-RNS state attached to a Context (constants and keys); see bfv.cu.
#pragma once

#include "context.hpp"

namespace lb {

struct BfvState {
    // filled by bfv_setup
};

}  // namespace lb
