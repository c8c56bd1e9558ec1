// Drop-in umbrella for code written against the reference's header-only API
// (proj/include/anvil/anvil.hpp). Including this instead of "anvil/anvil.hpp"
// and linking libfireiron_b200.so keeps every anvil:: call site compiling;
// anvil::run now executes on the B200 instead of the CPU model.
#pragma once

#include "fireiron/backend.hpp"
#include "fireiron/decomp.hpp"
#include "fireiron/error.hpp"
#include "fireiron/exec.hpp"
#include "fireiron/index_expr.hpp"
#include "fireiron/matrix.hpp"
#include "fireiron/program.hpp"
#include "fireiron/script.hpp"
#include "fireiron/types.hpp"

namespace anvil = fireiron;
