// Reference-compatible include path (perfseer/executor.hpp) for code written
// against the reference API; the declarations live in ps_executor.hpp.
#pragma once
#include "../ps_executor.hpp"
