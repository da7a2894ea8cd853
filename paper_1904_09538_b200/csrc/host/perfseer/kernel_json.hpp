// Reference-compatible include path (perfseer/kernel_json.hpp) for code written
// against the reference API; the declarations live in ps_json.hpp.
#pragma once
#include "../ps_json.hpp"
