// Thread-local error channel of the C ABI.
#pragma once

#include <string>

namespace fireiron::rt {

int set_error(int status, const std::string& msg);
void clear_error();
int device_sm_count();

}  // namespace fireiron::rt
