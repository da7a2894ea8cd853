// Reference-compatible include path (perfseer/ir.hpp) for code written
// against the reference API; the declarations live in ps_ir.hpp.
#pragma once
#include "../ps_ir.hpp"
