"""TEST INFRASTRUCTURE ONLY (see oracle/oracle.h). Not part of the product."""
