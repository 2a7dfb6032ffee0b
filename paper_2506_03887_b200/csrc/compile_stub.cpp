// compile_stub.cpp — placeholder until the host compile pipeline lands.
#include "gm_internal.hpp"
namespace pre3 {
Automaton CompileGrammar(const std::string&, bool, bool) {
  throw Error(GM_ERR_USAGE, "gm_automaton_compile: grammar compiler not built yet; load a P3DPDA file");
}
}  // namespace pre3
