// Host-side helpers shared by the C-ABI translation units.
#pragma once

#include <cuda_runtime.h>

#include "../../include/gfb.h"

namespace gfb {

int set_error(int code, const char *msg);
int check_launch(const char *what);
int sm_count();

}  // namespace gfb
