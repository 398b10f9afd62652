// Shared helpers between the setup and solver halves of the C ABI.
#pragma once

#include <string>

namespace dgb {
// Stores the message returned by dgb_last_message() on this thread.
void set_message(const std::string& s);
}  // namespace dgb
