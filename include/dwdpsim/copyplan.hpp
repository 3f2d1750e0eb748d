// Drop-in for /root/reference/proj/include/dwdpsim/copyplan.hpp: the reference's
// namespace dwdpsim API for this header, served by the libdwdp.so adapter.
#pragma once
#include "../dwdp.hpp"
