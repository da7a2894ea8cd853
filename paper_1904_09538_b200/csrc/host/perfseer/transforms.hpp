// Reference-compatible include path (perfseer/transforms.hpp) for code written
// against the reference API; the declarations live in ps_transforms.hpp.
#pragma once
#include "../ps_transforms.hpp"
