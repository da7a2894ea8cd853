// Reference-compatible include path (perfseer/features.hpp) for code written
// against the reference API; the declarations live in ps_features.hpp.
#pragma once
#include "../ps_features.hpp"
