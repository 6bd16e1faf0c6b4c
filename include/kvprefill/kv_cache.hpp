// kvprefill/kv_cache.hpp -- forwarding header so reference client code keeps its include line
// (`#include "kvprefill/kv_cache.hpp"`, reference proj/include/kvprefill/kv_cache.hpp) and gets the
// B200 drop-in: every name it declares lives in kvprefill_b200/kvprefill.hpp.
#pragma once
#include "../kvprefill_b200/kvprefill.hpp"
