// kvprefill/kvprefill.hpp -- forwarding header so reference client code keeps its include line
// (`#include "kvprefill/kvprefill.hpp"`, reference proj/include/kvprefill/kvprefill.hpp) and gets the
// B200 drop-in: every name it declares lives in kvprefill_b200/kvprefill.hpp.
#pragma once
#include "../kvprefill_b200/kvprefill.hpp"
