// kvprefill/lookup_table.hpp -- forwarding header (reference proj/include/kvprefill/
// lookup_table.hpp): PartitionLookupTable / interpolate_partition / partition_from_table are
// in kvprefill_b200/kvprefill.hpp, the JSON save/load in kvprefill_b200/table_io.hpp (needs
// nlohmann/json on the include path, as the reference's does).
#pragma once
#include "../kvprefill_b200/kvprefill.hpp"
#include "../kvprefill_b200/table_io.hpp"
