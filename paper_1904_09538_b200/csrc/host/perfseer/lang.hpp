// Reference-compatible include path (perfseer/lang.hpp) for code written
// against the reference API; the declarations live in ps_lang.hpp.
#pragma once
#include "../ps_lang.hpp"
